// Static-budget baselines (colbandit/baselines.py:49-86, doc_uniform / doc_top_margin): each row buys a
// fixed set of cells, and rows are ranked by the exactly rounded sum of the cells they bought
// (_ranked_by_partial_sum, baselines.py:38-41, math.fsum). The cell values come from the float64 cell
// kernel; this kernel gathers each row's chosen cells and sums them exactly (CPython msum semantics,
// Expansion in common.cuh), one thread per row. The ranking is the device Top-K on the sums.
#include "common.cuh"

namespace cbx {

constexpr int PS_CAP = 24;  // partials: far beyond what sums of <= 64 cells in [-1e3, 1e3] can need

__global__ void row_partial_fsum_kernel(const double* __restrict__ cells, int64_t ld, const int32_t* __restrict__ cols,
                                        int64_t n_rows, int b, double* __restrict__ sums, int* __restrict__ status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  Expansion<PS_CAP> ex;
  ex.clear();
  bool ok = true;
  for (int j = 0; j < b; ++j) ok &= ex.add(cells[i * ld + cols[i * b + j]]);
  if (!ok) atomicOr(status, 1);
  sums[i] = ex.round();
}

}  // namespace cbx

using namespace cbx;

extern "C" {

int cbx_row_partial_fsum(const double* cells, int64_t ld, const int32_t* cols, int64_t n_rows, int cells_per_row,
                         double* sums, int* status, void* stream) {
  if (n_rows < 0 || cells_per_row < 0 || ld < cells_per_row) return fail(CBX_EINVAL, "partial fsum: bad sizes");
  if (n_rows == 0) return CBX_OK;
  if (!cells || !sums || !status || (cells_per_row > 0 && !cols)) return fail(CBX_EINVAL, "partial fsum: NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  row_partial_fsum_kernel<<<(unsigned)((n_rows + 127) / 128), 128, 0, st>>>(cells, ld, cols, n_rows, cells_per_row,
                                                                          sums, status);
  CBX_LAUNCH_CHECK("row_partial_fsum_kernel launch");
  return CBX_OK;
}

}  // extern "C"
