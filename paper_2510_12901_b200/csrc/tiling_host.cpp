// simuli_build_tiles: automated LiDAR tiling (host, once per sensor definition).
//
// Proc. ElevationTiling (§3.3) with the DESIGN.md §3 A8
// readings, the ray table (A5), the tile -> ray CSR, and the dense ray mask + summed-area
// table used by ray-based culling (Proc. RayOccupancyCount P:524-542; A10).
// Float32 values that the interface defines (boundaries, ray angles, tile maps) are
// produced by fixed float32 operation sequences (no FMA contraction: this file is built
// with -ffp-contract=off) so the device kernels and any independent implementation of
// the same definitions agree bit-for-bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "abi_util.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;

// floor(u) clamped to [0, n-1]; NaN / negative -> 0 (shared rule of every float tile map)
inline int32_t clamp_floor(float u, int32_t n) {
  if (!(u >= 0.0f)) return 0;
  if (u >= static_cast<float>(n)) return n - 1;
  return std::min<int32_t>(static_cast<int32_t>(std::floor(u)), n - 1);
}

struct TileMaps {
  std::vector<float> bounds;     // n_phi + 1
  std::vector<float> row_scale;  // n_phi
  int32_t n_phi = 1, n_theta = 1, rows_per_tile = 8, az_cells = 1600;
  float pi_f = 0, two_pi_f = 0, az_tile_scale = 0, az_cell_scale = 0;

  // elevation tile = number of interior boundaries <= w
  int32_t elev_tile(float w) const {
    auto first = bounds.begin() + 1, last = bounds.begin() + n_phi;  // interior [1, n_phi-1]
    return static_cast<int32_t>(std::upper_bound(first, last, w) - first);
  }
  int32_t az_index(float phi, float scale, int32_t n) const {
    float a = phi + pi_f;
    float u = a * scale;
    return clamp_floor(u, n);
  }
  int32_t az_tile(float phi) const { return az_index(phi, az_tile_scale, n_theta); }
  int32_t az_cell(float phi) const { return az_index(phi, az_cell_scale, az_cells); }
  int32_t dense_row(float w) const {
    int32_t e = elev_tile(w);
    float a = w - bounds[e];
    float u = a * row_scale[e];
    return e * rows_per_tile + clamp_floor(u, rows_per_tile);
  }
};

// Partition of beams into elevation tiles (Proc. ElevationTiling lines 1-11, A8).
// Returns the tile index of every beam, tiles numbered 0..n_parts-1 by elevation.
std::vector<int32_t> equalised_partition(const std::vector<float>& elev, int32_t n_az, int32_t n_phi, int32_t bins,
                                         int32_t* n_parts) {
  const size_t B = elev.size();
  std::vector<int32_t> part(B, 0);
  const double lo = *std::min_element(elev.begin(), elev.end());
  const double hi = *std::max_element(elev.begin(), elev.end());
  if (!(hi > lo)) {  // all beams at one elevation: a single tile
    *n_parts = 1;
    return part;
  }
  // histogram of per-ray elevations: every beam contributes its n_az rays
  std::vector<int32_t> bin_of(B);
  std::vector<int64_t> hist(bins, 0);
  for (size_t b = 0; b < B; ++b) {
    int32_t k = static_cast<int32_t>(std::floor((static_cast<double>(elev[b]) - lo) / (hi - lo) * bins));
    bin_of[b] = std::min(k, bins - 1);
    hist[bin_of[b]] += n_az;
  }
  // normalised CDF crossing integer b  <=>  cum * n_phi >= b * total (exact); at most one
  // crossing per bin; the crossing bin closes the current tile.
  const int64_t total = static_cast<int64_t>(B) * n_az;
  std::vector<int32_t> crossing_bins;
  int64_t cum = 0, next = 1;
  for (int32_t i = 0; i < bins; ++i) {
    cum += hist[i];
    if (cum * n_phi >= next * total) {
      crossing_bins.push_back(i);
      ++next;
    }
  }
  // raw tile of a bin = number of crossings strictly before it; then drop empty tiles
  std::vector<int32_t> raw(B);
  for (size_t b = 0; b < B; ++b)
    raw[b] = static_cast<int32_t>(std::lower_bound(crossing_bins.begin(), crossing_bins.end(), bin_of[b]) -
                                  crossing_bins.begin());
  std::vector<int32_t> used(raw);
  std::sort(used.begin(), used.end());
  used.erase(std::unique(used.begin(), used.end()), used.end());
  for (size_t b = 0; b < B; ++b)
    part[b] = static_cast<int32_t>(std::lower_bound(used.begin(), used.end(), raw[b]) - used.begin());
  *n_parts = static_cast<int32_t>(used.size());
  return part;
}

}  // namespace

extern "C" int32_t simuli_build_tiles(const simuli_lidar* lidar, const simuli_tiling_params* prm,
                                      simuli_tiling* out) {
  using simuli::set_error;
  simuli::clear_error();
  SIMULI_REQUIRE(lidar && prm && out, "simuli_build_tiles: NULL argument");
  SIMULI_REQUIRE(lidar->n_beams >= 1 && lidar->beam_elevation_rad, "n_beams must be >= 1 with elevations");
  SIMULI_REQUIRE(lidar->n_azimuth >= 1, "n_azimuth must be >= 1");
  SIMULI_REQUIRE(lidar->spin_direction == 1 || lidar->spin_direction == -1, "spin_direction must be +-1");
  SIMULI_REQUIRE(prm->n_phi >= 1 && prm->max_rays_per_tile >= 1 && prm->hist_bins >= 1 && prm->cull_az_cells >= 1 &&
                     prm->cull_rows_per_tile >= 1,
                 "tiling parameters must be >= 1");
  SIMULI_REQUIRE(prm->n_phi <= prm->hist_bins, "tile count exceeds histogram resolution");
  const int32_t B = lidar->n_beams, A = lidar->n_azimuth;
  std::vector<float> elev(lidar->beam_elevation_rad, lidar->beam_elevation_rad + B);
  for (float e : elev) SIMULI_REQUIRE(std::fabs(static_cast<double>(e)) < kPi / 2, "beam elevation outside (-pi/2, pi/2)");

  int32_t n_parts = 1;
  std::vector<int32_t> part = equalised_partition(elev, A, prm->n_phi, prm->hist_bins, &n_parts);

  TileMaps tm;
  tm.n_phi = n_parts;
  tm.rows_per_tile = prm->cull_rows_per_tile;
  tm.az_cells = prm->cull_az_cells;
  tm.bounds.assign(n_parts + 1, 0.0f);
  tm.bounds.front() = *std::min_element(elev.begin(), elev.end());
  tm.bounds.back() = *std::max_element(elev.begin(), elev.end());
  std::vector<float> top(n_parts, -INFINITY), bottom(n_parts, INFINITY);
  std::vector<int32_t> beams_in(n_parts, 0);
  for (int32_t b = 0; b < B; ++b) {
    top[part[b]] = std::max(top[part[b]], elev[b]);
    bottom[part[b]] = std::min(bottom[part[b]], elev[b]);
    beams_in[part[b]]++;
  }
  for (int32_t k = 1; k < n_parts; ++k) {  // boundary in the gap between tiles k-1 and k
    const float below = top[k - 1], above = bottom[k];
    float mid = static_cast<float>((static_cast<double>(below) + static_cast<double>(above)) * 0.5);
    if (mid <= below) mid = above;
    tm.bounds[k] = mid;
  }
  tm.row_scale.resize(n_parts);
  for (int32_t k = 0; k < n_parts; ++k) {
    const double width = static_cast<double>(tm.bounds[k + 1]) - static_cast<double>(tm.bounds[k]);
    tm.row_scale[k] = width > 0.0 ? static_cast<float>(prm->cull_rows_per_tile / width) : 0.0f;
  }
  for (int32_t b = 0; b < B; ++b)
    if (tm.elev_tile(elev[b]) != part[b]) {
      set_error("internal: float32 boundaries do not reproduce the beam partition");
      return SIMULI_ERR_INVALID_ARGUMENT;
    }
  // lines 12-13: azimuth tiles from the max re-histogram count and M
  const int64_t h_max = static_cast<int64_t>(*std::max_element(beams_in.begin(), beams_in.end())) * A;
  int64_t n_theta = (h_max + prm->max_rays_per_tile - 1) / prm->max_rays_per_tile;
  n_theta = std::max<int64_t>(1, std::min<int64_t>(n_theta, A));
  tm.n_theta = static_cast<int32_t>(n_theta);
  tm.pi_f = static_cast<float>(kPi);
  tm.two_pi_f = static_cast<float>(kTwoPi);
  tm.az_tile_scale = static_cast<float>(static_cast<double>(tm.n_theta) / kTwoPi);
  tm.az_cell_scale = static_cast<float>(static_cast<double>(prm->cull_az_cells) / kTwoPi);

  const int32_t n_tiles = n_parts * tm.n_theta;
  const int32_t R = B * A;
  const int32_t rows = prm->cull_rows_per_tile * n_parts, cols = prm->cull_az_cells;

  // column azimuths / times (shared by all beams, A5)
  std::vector<float> col_phi(A), col_s(A);
  std::vector<int32_t> col_tile(A);
  for (int32_t j = 0; j < A; ++j) {
    double phi = static_cast<double>(lidar->azimuth_start_rad) +
                 static_cast<double>(lidar->spin_direction) * ((static_cast<double>(j) + 0.5) * (kTwoPi / A));
    if (phi >= kPi)
      phi -= kTwoPi;
    else if (phi < -kPi)
      phi += kTwoPi;
    col_phi[j] = static_cast<float>(phi);
    col_s[j] = static_cast<float>((static_cast<double>(j) + 0.5) / A);
    col_tile[j] = tm.az_tile(col_phi[j]);
  }
  std::vector<int32_t> ray_tile(R);
  std::vector<int32_t> tile_count(n_tiles, 0);
  int32_t max_in_tile = 0;
  for (int32_t b = 0; b < B; ++b)
    for (int32_t j = 0; j < A; ++j) {
      const int32_t t = part[b] * tm.n_theta + col_tile[j];
      ray_tile[b * A + j] = t;
      max_in_tile = std::max(max_in_tile, ++tile_count[t]);
    }

  out->n_phi = n_parts;
  out->n_theta = tm.n_theta;
  out->n_tiles = n_tiles;
  out->max_rays_in_tile = max_in_tile;
  out->sat_rows = rows + 1;
  out->sat_cols = cols + 1;
  out->n_rays = R;
  out->n_beams = B;
  out->n_azimuth = A;
  out->max_beams_per_elev_tile = *std::max_element(beams_in.begin(), beams_in.end());
  {
    std::vector<int32_t> cols_in(tm.n_theta, 0);
    for (int32_t j = 0; j < A; ++j) cols_in[col_tile[j]]++;
    out->max_cols_per_az_tile = *std::max_element(cols_in.begin(), cols_in.end());
  }
  out->pi_f = tm.pi_f;
  out->two_pi_f = tm.two_pi_f;
  out->az_tile_scale = tm.az_tile_scale;
  out->az_cell_scale = tm.az_cell_scale;

  const bool sizing = !out->elev_bounds && !out->cull_row_scale && !out->ray_az && !out->ray_el && !out->ray_s &&
                      !out->ray_tile && !out->tile_ray_offsets && !out->tile_rays && !out->sat &&
                      !out->elev_tile_beam_offsets && !out->elev_tile_beams && !out->az_tile_col_offsets &&
                      !out->az_tile_cols && !out->beam_el_sorted && !out->col_az_sorted;
  if (sizing) return SIMULI_OK;
  SIMULI_REQUIRE(out->elev_bounds && out->cull_row_scale && out->ray_az && out->ray_el && out->ray_s &&
                     out->ray_tile && out->tile_ray_offsets && out->tile_rays && out->sat &&
                     out->elev_tile_beam_offsets && out->elev_tile_beams && out->az_tile_col_offsets &&
                     out->az_tile_cols && out->beam_el_sorted && out->col_az_sorted,
                 "simuli_build_tiles: either all or none of the array pointers must be set");

  std::copy(tm.bounds.begin(), tm.bounds.end(), out->elev_bounds);
  std::copy(tm.row_scale.begin(), tm.row_scale.end(), out->cull_row_scale);
  for (int32_t b = 0; b < B; ++b)
    for (int32_t j = 0; j < A; ++j) {
      const int32_t r = b * A + j;
      out->ray_az[r] = col_phi[j];
      out->ray_el[r] = elev[b];
      out->ray_s[r] = col_s[j];
      out->ray_tile[r] = ray_tile[r];
    }
  // CSR tile -> rays (ray ids increasing within a tile)
  out->tile_ray_offsets[0] = 0;
  for (int32_t t = 0; t < n_tiles; ++t) out->tile_ray_offsets[t + 1] = out->tile_ray_offsets[t] + tile_count[t];
  std::vector<int32_t> cursor(out->tile_ray_offsets, out->tile_ray_offsets + n_tiles);
  for (int32_t r = 0; r < R; ++r) out->tile_rays[cursor[ray_tile[r]]++] = r;
  // CSR elevation tile -> beams, azimuth tile -> columns
  out->elev_tile_beam_offsets[0] = 0;
  for (int32_t k = 0; k < n_parts; ++k) out->elev_tile_beam_offsets[k + 1] = out->elev_tile_beam_offsets[k] + beams_in[k];
  std::vector<int32_t> bc(out->elev_tile_beam_offsets, out->elev_tile_beam_offsets + n_parts);
  for (int32_t b = 0; b < B; ++b) out->elev_tile_beams[bc[part[b]]++] = b;
  std::vector<int32_t> cols_in(tm.n_theta, 0);
  for (int32_t j = 0; j < A; ++j) cols_in[col_tile[j]]++;
  out->az_tile_col_offsets[0] = 0;
  for (int32_t c = 0; c < tm.n_theta; ++c) out->az_tile_col_offsets[c + 1] = out->az_tile_col_offsets[c] + cols_in[c];
  std::vector<int32_t> cc(out->az_tile_col_offsets, out->az_tile_col_offsets + tm.n_theta);
  for (int32_t j = 0; j < A; ++j) out->az_tile_cols[cc[col_tile[j]]++] = j;
  // ascending beam elevations / column azimuths: the exact culling's binary searches (A32)
  std::copy(elev.begin(), elev.end(), out->beam_el_sorted);
  std::sort(out->beam_el_sorted, out->beam_el_sorted + B);
  std::copy(col_phi.begin(), col_phi.end(), out->col_az_sorted);
  std::sort(out->col_az_sorted, out->col_az_sorted + A);
  // dense ray mask (cells hit by >= 1 ray) -> summed-area table, zero first row/column
  std::vector<uint8_t> mask(static_cast<size_t>(rows) * cols, 0);
  std::vector<int32_t> beam_row(B);
  for (int32_t b = 0; b < B; ++b) beam_row[b] = tm.dense_row(elev[b]);
  for (int32_t j = 0; j < A; ++j) {
    const int32_t cell = tm.az_cell(col_phi[j]);
    for (int32_t b = 0; b < B; ++b) mask[static_cast<size_t>(beam_row[b]) * cols + cell] = 1;
  }
  const int32_t sc = cols + 1;
  std::fill(out->sat, out->sat + static_cast<size_t>(rows + 1) * sc, 0);
  for (int32_t i = 0; i < rows; ++i) {
    int32_t run = 0;  // prefix along the row, then add the row above
    for (int32_t j = 0; j < cols; ++j) {
      run += mask[static_cast<size_t>(i) * cols + j];
      out->sat[static_cast<size_t>(i + 1) * sc + (j + 1)] = out->sat[static_cast<size_t>(i) * sc + (j + 1)] + run;
    }
  }
  return SIMULI_OK;
}
