// K2 bandit kernels for __half tokens (see bandit_impl.cuh): the dispatchers, the warm-up pre-pass and the
// layouts of rows above 512 bytes; the other layouts live in bandit_f16_g16.cu and bandit_f16_g8_g32.cu so the
// instantiations compile in parallel. Built with -fmad=false like every bandit*.cu unit.
#include "bandit_impl.cuh"

namespace cbx {
template int launch_bandit<__half, 32, 2>(const BanditParams&, int64_t, size_t, cudaStream_t);
template int launch_bandit<__half, 32, 4>(const BanditParams&, int64_t, size_t, cudaStream_t);
template int dispatch_bandit<__half>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
template int dispatch_warm<__half>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);
}  // namespace cbx
