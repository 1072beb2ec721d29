"""B200-native MorphServe serving hot path (arXiv 2506.02006).

Layers: CUDA kernels + C ABI (csrc/, include/morphserve.h, lib/libmorphserve.so),
C++ host runtime (csrc/host/, lib/libmorphserve_host.so, _core), and the
drop-in ``morphsim`` Python API (paper_2506_02006_b200.morphsim).
"""
