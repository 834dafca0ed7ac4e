"""B200-native SimULi forward sensor-rendering hot path (arXiv 2510.12901).

libsimuli.so (paper_2510_12901_b200/csrc, hand-written CUDA for sm_100a) behind the C ABI
of include/simuli.h; ``simuli`` is the thin ctypes binding; ``synth`` holds the seeded
synthetic inputs.  Nothing here imports the test oracle (oracle/).
"""
__all__ = ["simuli", "synth", "build"]
