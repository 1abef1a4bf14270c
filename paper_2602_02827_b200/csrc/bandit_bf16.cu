// K2 bandit kernels for __nv_bfloat16 tokens (see bandit_impl.cuh): one translation unit per dtype so the
// instantiations compile in parallel. Built with -fmad=false like every bandit*.cu unit.
#include "bandit_impl.cuh"

namespace cbx {
template int dispatch_bandit<__nv_bfloat16>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
template int dispatch_warm<__nv_bfloat16>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);
}  // namespace cbx
