"""B200-native buffer-coherence path of Celerity instruction-graph scheduling
(arXiv 2503.10516): C++ scheduler + sm_100a kernels behind the C-ABI in
include/cel.h; `cel` is the ctypes binding."""
