// Device-side building blocks of libsimuli (sm_100a).  Internal header.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/simuli.h"
#include "abi_util.h"

// Checked builds (SIMULI_EXTRA_NVCC=-DSIMULI_CHECKED, scripts/checked_run.sh): device-side
// bounds / invariant assertions on the kernels' computed indices -- the substitute for
// compute-sanitizer, which is closed on the GPU pool.  A failed check prints the kernel's
// file:line and the operands, then traps (the launch fails with an illegal-instruction
// error the caller sees).  Compiled out otherwise.
#ifdef SIMULI_CHECKED
#include <cstdio>
#define SIMULI_CHECK(cond, a, b)                                                                            \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("SIMULI_CHECK failed %s:%d: %s (%lld, %lld) block %d thread %d\n", __FILE__, __LINE__, #cond, \
             (long long)(a), (long long)(b), (int)blockIdx.x, (int)threadIdx.x);                          \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define SIMULI_CHECK(cond, a, b) \
  do {                           \
  } while (0)
#endif

namespace simuli {

// Programmatic dependent launch (sm_90+): the forward path's kernels are launched with
// programmatic stream serialization, so kernel k + 1's CTAs are scheduled while kernel k's
// last CTAs finish (hiding the launch gap between dependent kernels on one stream).  Every
// such kernel starts with pdl_wait() -- it blocks until the previous grid on the stream has
// completed and its writes are visible, so nothing before it may read what that grid
// produced -- then pdl_trigger() lets the next grid launch once all CTAs of this one have
// started.  Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("SIMULI_PDL");  // tuning / A-B only: 0 = plain launches
    return !(v && v[0] == '0');
  }();
  return on;
}

// kernel<<<grid, block, smem, st>>>(args...) with programmatic stream serialization
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  if (!pdl_enabled()) {
    kernel<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// status of the last kernel launch as a libsimuli error code (with the CUDA message)
inline int32_t launch_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return SIMULI_ERR_CUDA;
  }
  return SIMULI_OK;
}

constexpr int kRecordFloats = 20;  // mu 3, M 9, opacity 1, f 3, box 4  (80 B)

// Sensor pose interpolation between start and end (A4): t(s) = t0 + s dt,
// q(s) = q0 * [cos(s theta/2), sin(s theta/2) axis] (slerp on the shortest arc, identical
// to R0 Exp(s Log(R0^T R1))).  Built on the host in double.
struct PoseInterpF {
  float q0[4];  // normalised
  float axis[3];
  float half_theta;
  float t0[3], dt[3];
  int same;  // start == end: R(s) = R0, t(s) = t0 exactly
};
struct PoseInterpD {
  double q0[4];
  double axis[3];
  double half_theta;
  double t0[3], dt[3];
  int same;
};

PoseInterpD make_pose_interp_d(const simuli_pose& a, const simuli_pose& b);
PoseInterpF make_pose_interp_f(const PoseInterpD& d);

template <typename T>
__device__ __forceinline__ void quat_rot(const T q[4], T R[9]) {
  const T w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = T(1) - T(2) * (y * y + z * z);
  R[1] = T(2) * (x * y - w * z);
  R[2] = T(2) * (x * z + w * y);
  R[3] = T(2) * (x * y + w * z);
  R[4] = T(1) - T(2) * (x * x + z * z);
  R[5] = T(2) * (y * z - w * x);
  R[6] = T(2) * (x * z - w * y);
  R[7] = T(2) * (y * z + w * x);
  R[8] = T(1) - T(2) * (x * x + y * y);
}

__device__ __forceinline__ void pose_at(const PoseInterpF& P, float s, float R[9], float t[3]) {
  float q[4];
  if (P.same) {
    q[0] = P.q0[0]; q[1] = P.q0[1]; q[2] = P.q0[2]; q[3] = P.q0[3];
  } else {
    float sn, cs;
    sincosf(s * P.half_theta, &sn, &cs);
    const float b[4] = {cs, sn * P.axis[0], sn * P.axis[1], sn * P.axis[2]};
    const float* a = P.q0;
    q[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    q[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    q[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    q[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  }
  quat_rot(q, R);
  t[0] = P.t0[0] + s * P.dt[0];
  t[1] = P.t0[1] + s * P.dt[1];
  t[2] = P.t0[2] + s * P.dt[2];
}

__device__ __forceinline__ void pose_at_d(const PoseInterpD& P, double s, double R[9], double t[3]) {
  double q[4];
  if (P.same) {
    q[0] = P.q0[0]; q[1] = P.q0[1]; q[2] = P.q0[2]; q[3] = P.q0[3];
  } else {
    double sn, cs;
    sincos(s * P.half_theta, &sn, &cs);
    const double b[4] = {cs, sn * P.axis[0], sn * P.axis[1], sn * P.axis[2]};
    const double* a = P.q0;
    q[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    q[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    q[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    q[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
  }
  quat_rot(q, R);
  t[0] = P.t0[0] + s * P.dt[0];
  t[1] = P.t0[1] + s * P.dt[1];
  t[2] = P.t0[2] + s * P.dt[2];
}

// floor(u) clamped to [0, n-1]; NaN / negative -> 0 (the shared float32 tile-map rule)
__device__ __forceinline__ int clamp_floor(float u, int n) {
  if (!(u >= 0.0f)) return 0;
  if (u >= (float)n) return n - 1;
  return min((int)floorf(u), n - 1);
}

// azimuth -> index with correctly rounded float32 ops: floor((phi + pi_f) * scale)
__device__ __forceinline__ int az_index(float phi, float pi_f, float scale, int n) {
  return clamp_floor(__fmul_rn(__fadd_rn(phi, pi_f), scale), n);
}

// Circular index run [start, start+len) covered by the azimuth interval [lo, hi] (floats
// shifted by 2 pi_f, never the rays; A12).
__device__ __forceinline__ void az_run(float lo, float hi, float pi_f, float two_pi_f, float scale, int n,
                                       int* start, int* len) {
  if (__fsub_rn(hi, lo) >= two_pi_f) {
    *start = 0;
    *len = n;
    return;
  }
  const int ia = az_index(fmaxf(lo, -pi_f), pi_f, scale, n);
  const int ib = az_index(fminf(hi, pi_f), pi_f, scale, n);
  if (lo < -pi_f) {
    const int ic = az_index(__fadd_rn(lo, two_pi_f), pi_f, scale, n);
    if (ic <= ib + 1) { *start = 0; *len = n; }
    else { *start = ic; *len = (n - ic) + ib + 1; }
  } else if (hi > pi_f) {
    const int id = az_index(__fsub_rn(hi, two_pi_f), pi_f, scale, n);
    if (id >= ia - 1) { *start = 0; *len = n; }
    else { *start = ia; *len = (n - ia) + id + 1; }
  } else {
    *start = ia;
    *len = ib - ia + 1;
  }
}

// ray (a, b) inside box [lo_a, hi_a] x [lo_b, hi_b] with the LiDAR azimuth wrap rules (A12)
__device__ __forceinline__ bool in_box_wrap(float lo_a, float hi_a, float lo_b, float hi_b, float a, float b,
                                            float pi_f, float two_pi_f) {
  if (!(lo_b <= b && b <= hi_b)) return false;
  if (__fsub_rn(hi_a, lo_a) >= two_pi_f) return true;
  if (lo_a <= a && a <= hi_a) return true;
  if (lo_a < -pi_f && __fadd_rn(lo_a, two_pi_f) <= a) return true;
  if (hi_a > pi_f && a <= __fsub_rn(hi_a, two_pi_f)) return true;
  return false;
}

// Degree-<=3 real SH (3DGS constants), coefficients [(deg+1)^2][3]
__device__ __forceinline__ void sh_eval(const float* __restrict__ sh, int degree, float x, float y, float z,
                                        float out[3]) {
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
  float b[16];
  b[0] = C0;
  int nb = 1;
  if (degree >= 1) {
    b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    nb = 4;
  }
  if (degree >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = 1.0925484305920792f * x * y;
    b[5] = -1.0925484305920792f * y * z;
    b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    b[7] = -1.0925484305920792f * x * z;
    b[8] = 0.5462742152960396f * (xx - yy);
    nb = 9;
  }
  if (degree >= 3) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    b[10] = 2.890611442640554f * x * y * z;
    b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
    nb = 16;
  }
  float r0 = 0.f, r1 = 0.f, r2 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k < nb) {
      r0 = fmaf(b[k], __ldg(sh + 3 * k + 0), r0);
      r1 = fmaf(b[k], __ldg(sh + 3 * k + 1), r1);
      r2 = fmaf(b[k], __ldg(sh + 3 * k + 2), r2);
    }
  }
  out[0] = r0; out[1] = r1; out[2] = r2;
}

// The 16 real SH basis values of degree <= 3 at the unit direction (x, y, z)
__device__ __forceinline__ void sh_basis3(float x, float y, float z, float b[16]) {
  const float xx = x * x, yy = y * y, zz = z * z;
  b[0] = 0.28209479177387814f;
  b[1] = -0.4886025119029199f * y;
  b[2] = 0.4886025119029199f * z;
  b[3] = -0.4886025119029199f * x;
  b[4] = 1.0925484305920792f * x * y;
  b[5] = -1.0925484305920792f * y * z;
  b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
  b[7] = -1.0925484305920792f * x * z;
  b[8] = 0.5462742152960396f * (xx - yy);
  b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
  b[10] = 2.890611442640554f * x * y * z;
  b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
  b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
  b[14] = 1.445305721320277f * z * (xx - yy);
  b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// Eq. 1 literally (A30): one particle's SH features at a ray direction whose
// basis b (sh_basis3) the caller computed once per ray; ncoef = (degree + 1)^2 coefficients
// [ncoef][3], summed in coefficient order.  Degree 3 reads the 192-byte block as 12 float4.
__device__ __forceinline__ void sh_dot(const float* __restrict__ sh, int ncoef, const float b[16], float f[3]) {
  float acc[3] = {0.f, 0.f, 0.f};
  if (ncoef == 16) {
    const float4* s4 = reinterpret_cast<const float4*>(sh);
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const float4 v4 = __ldg(s4 + c);
      const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[(4 * c + j) % 3] = fmaf(b[(4 * c + j) / 3], v[j], acc[(4 * c + j) % 3]);
    }
  } else {
    for (int k = 0; k < ncoef; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = fmaf(b[k], __ldg(sh + 3 * k + c), acc[c]);
  }
  f[0] = acc[0]; f[1] = acc[1]; f[2] = acc[2];
}

// The same for degree 3 from a 192-byte block already staged (e.g. in shared memory).
__device__ __forceinline__ void sh_dot16(const float4* s4, const float b[16], float f[3]) {
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    const float4 v4 = s4[c];
    const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[(4 * c + j) % 3] = fmaf(b[(4 * c + j) / 3], v[j], acc[(4 * c + j) % 3]);
  }
  f[0] = acc[0]; f[1] = acc[1]; f[2] = acc[2];
}

// Ray in double, split into float hi + lo parts for the compensated response.
struct RayF {
  float o_hi[3], o_lo[3], d_hi[3], d_lo[3];
};

__device__ __forceinline__ void split_ray(const double o[3], const double d[3], RayF& r) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.o_hi[k] = (float)o[k];
    r.o_lo[k] = (float)(o[k] - (double)r.o_hi[k]);
    r.d_hi[k] = (float)d[k];
    r.d_lo[k] = (float)(d[k] - (double)r.d_hi[k]);
  }
}

// 3D particle response at tau_max in canonical space, computed without the
// cancellation of |o - mu| ~ 1e2 m against particle scales ~ 1e-2 m:
//   p = o - mu (exact two-sum + o_lo), t = p.d, p_perp = p - t d (FMA; any error of t lies
//   along d and cancels below), a = M p_perp, d' = M d,
//   tau = -t - (a.d')/|d'|^2,  delta^2 = |d' x a|^2 / |d'|^2   (= |(d'/|d'|) x M(o-mu)|^2)
__device__ __forceinline__ void response(const RayF& r, const float mu[3], const float M[9], float* tau,
                                         float* delta2) {
  float ph[3], pl[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a = r.o_hi[k], b = -mu[k];
    const float s = __fadd_rn(a, b);
    const float bb = __fsub_rn(s, a);
    const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    ph[k] = s;
    pl[k] = err + r.o_lo[k];
  }
  const float t = ph[0] * r.d_hi[0] + ph[1] * r.d_hi[1] + ph[2] * r.d_hi[2];
  float pp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pp[k] = fmaf(-t, r.d_hi[k], ph[k]) + fmaf(-t, r.d_lo[k], pl[k]);
  float a[3], dd[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    a[k] = M[3 * k] * pp[0] + M[3 * k + 1] * pp[1] + M[3 * k + 2] * pp[2];
    dd[k] = M[3 * k] * r.d_hi[0] + M[3 * k + 1] * r.d_hi[1] + M[3 * k + 2] * r.d_hi[2];
  }
  const float dd2 = dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2];
  const float inv = 1.0f / dd2;
  *tau = -t - (a[0] * dd[0] + a[1] * dd[1] + a[2] * dd[2]) * inv;
  const float cx = dd[1] * a[2] - dd[2] * a[1];
  const float cy = dd[2] * a[0] - dd[0] * a[2];
  const float cz = dd[0] * a[1] - dd[1] * a[0];
  *delta2 = (cx * cx + cy * cy + cz * cz) * inv;
}

__device__ __forceinline__ float raydrop_prob(float z1, float z2) {
  const float z = z1 - z2;
  if (z >= 0.0f) {
    const float e = expf(-z);
    return e / (1.0f + e);
  }
  return 1.0f / (1.0f + expf(z));
}

}  // namespace simuli
