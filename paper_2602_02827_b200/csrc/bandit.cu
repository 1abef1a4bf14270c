// K2 — Col-Bandit adaptive loop (placeholder until the persistent kernel lands).
#include "common.cuh"

using namespace cbx;

extern "C" {
size_t cbx_bandit_state_bytes(int64_t total_rows, int32_t max_t) { return 0; }
int cbx_bandit_run(const cbx_batch*, const double*, int64_t, int32_t, const cbx_bandit_run_desc*, int64_t,
                   const double*, const double*, const int32_t*, void*, size_t, int32_t*, int32_t, int32_t*,
                   int32_t*, double*, cbx_bandit_out*, void*) {
  return fail(CBX_EINTERNAL, "bandit kernel not built yet");
}
}
