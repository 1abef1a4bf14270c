// K2 bandit kernels for __nv_bfloat16 tokens, rows of up to 128 bytes and of 257-512 bytes (d = 256: cfg5).
// Built with -fmad=false like every bandit*.cu unit.
#include "bandit_impl.cuh"

namespace cbx {
template int launch_bandit<__nv_bfloat16, 8, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);
template int launch_bandit<__nv_bfloat16, 32, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);
}  // namespace cbx
