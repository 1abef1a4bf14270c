// K2 bandit kernels for __nv_bfloat16 tokens, rows of 129-256 bytes (d = 128: the BASELINE configs' layout).
// Built with -fmad=false like every bandit*.cu unit.
#include "bandit_impl.cuh"

namespace cbx {
template int launch_bandit<__nv_bfloat16, 16, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);
}  // namespace cbx
