// K0 — float64-exact MaxSim cells and scores on the CUDA cores.
//
// Replaces MaxSimOracle.row_values / maxsim / full_score
// (colbandit/oracle.py:205-227): cell H[i, t] = max_j <e_ij, q_t> summed in
// float64 from exact products (fp16/bf16/fp32 products are exact in
// float64; for fp16/bf16 unit vectors the sums are exact too, so any
// accumulation order reproduces the reference bit for bit — SURVEY F3), then
// floored at 0 under clamp_negative (oracle.py:65-66). The row score is the
// exactly rounded sum of the row (math.fsum semantics, oracle.py:225).
//
// Used for fp32/fp64 inputs (where TF32 tensor cores would break the 1e-5
// tolerance), for the drop-in oracle's cell accessors and for full_rerank.
// One CTA per document; the query lives in shared memory (float for
// 16/32-bit inputs, double for fp64); warps stride over document tokens and
// lanes over query tokens.
#include "common.cuh"

namespace cbx {

constexpr int EX_THREADS = 256;
constexpr int EX_WARPS = EX_THREADS / 32;

template <typename T>
using ExStore = typename std::conditional<std::is_same<T, double>::value, double, float>::type;

__device__ __forceinline__ int64_t query_of_doc(const int64_t* __restrict__ q_doc_off, int64_t nq, int64_t doc) {
  // last q with q_doc_off[q] <= doc
  int64_t lo = 0, hi = nq;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(q_doc_off + mid) <= doc) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <typename T>
__global__ void __launch_bounds__(EX_THREADS)
    maxsim_exact_kernel(const T* __restrict__ q_tokens, const int64_t* __restrict__ q_tok_off,
                        const T* __restrict__ d_tokens, const int64_t* __restrict__ d_tok_off,
                        const int64_t* __restrict__ q_doc_off, int64_t n_queries, int64_t n_docs, int dim,
                        int clamp_negative, double* __restrict__ cells, int64_t ld, double* __restrict__ scores64,
                        float* __restrict__ scores32) {
  using S = ExStore<T>;
  extern __shared__ __align__(16) uint8_t ex_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dp = dim + 1;  // padded row stride: lanes read distinct banks
  for (int64_t doc = blockIdx.x; doc < n_docs; doc += gridDim.x) {
    const int64_t q = query_of_doc(q_doc_off, n_queries, doc);
    const int64_t qt0 = q_tok_off[q];
    const int lq = (int)(q_tok_off[q + 1] - qt0);
    const int64_t j0 = d_tok_off[doc], j1 = d_tok_off[doc + 1];
    S* qs = reinterpret_cast<S*>(ex_smem);
    double* wmax = reinterpret_cast<double*>(ex_smem + align_up_dev(sizeof(S) * (size_t)lq * dp, 16));
    __syncthreads();
    for (int i = threadIdx.x; i < lq * dim; i += EX_THREADS) {
      int t = i / dim, k = i - t * dim;
      qs[t * dp + k] = (S)Elem<T>::to_d(q_tokens[(qt0 + t) * dim + k]);
    }
    __syncthreads();
    for (int tb = 0; tb < lq; tb += 32) {
      const int t = tb + lane;
      double best = clamp_negative ? 0.0 : -INFINITY;
      if (t < lq) {
        const S* qrow = qs + t * dp;
        for (int64_t j = j0 + warp; j < j1; j += EX_WARPS) {
          const T* e = d_tokens + j * dim;
          double acc = 0.0;
          for (int k = 0; k < dim; ++k) acc = fma(Elem<T>::to_d(__ldg(e + k)), (double)qrow[k], acc);
          best = acc > best ? acc : best;
        }
      }
      wmax[warp * 32 + lane] = best;
      __syncthreads();
      if (warp == 0 && t < lq) {
        double m = wmax[lane];
        for (int w = 1; w < EX_WARPS; ++w) m = wmax[w * 32 + lane] > m ? wmax[w * 32 + lane] : m;
        wmax[EX_WARPS * 32 + t] = m;  // row staging for the score
        if (cells) cells[doc * ld + t] = m;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0 && (scores64 || scores32)) {
      const double* row = wmax + EX_WARPS * 32;
      Expansion<8> ex;
      ex.clear();
      for (int t = 0; t < lq; ++t) ex.add(row[t]);
      double s = ex.round();
      if (scores64) scores64[doc] = s;
      if (scores32) scores32[doc] = (float)s;
    }
  }
}

template <typename T>
static int launch_exact_t(const cbx_batch* b, double* cells, int64_t ld, double* s64, float* s32, cudaStream_t st) {
  using S = ExStore<T>;
  size_t smem = align_up(sizeof(S) * (size_t)b->max_lq * (b->dim + 1), 16) +
                sizeof(double) * (EX_WARPS * 32 + std::max<int64_t>(b->max_lq, 32) + 32);
  if (smem > 227 * 1024) return fail(CBX_EINVAL, "exact scorer: query too large for shared memory");
  CBX_CUDA_CHECK(cudaFuncSetAttribute(maxsim_exact_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = (int)std::min<int64_t>(b->n_docs, (int64_t)sm_count() * 8);
  maxsim_exact_kernel<T><<<grid, EX_THREADS, smem, st>>>(
      static_cast<const T*>(b->q_tokens), b->q_tok_off, static_cast<const T*>(b->d_tokens), b->d_tok_off,
      b->q_doc_off, b->n_queries, b->n_docs, b->dim, b->clamp_negative, cells, ld, s64, s32);
  CBX_LAUNCH_CHECK("maxsim_exact_kernel launch");
  return CBX_OK;
}

int launch_maxsim_exact(const cbx_batch* b, double* cells, int64_t ld, double* s64, float* s32, cudaStream_t st) {
  if (b->n_docs == 0) return CBX_OK;
  switch (b->dtype) {
    case CBX_F32: return launch_exact_t<float>(b, cells, ld, s64, s32, st);
    case CBX_F64: return launch_exact_t<double>(b, cells, ld, s64, s32, st);
    case CBX_F16: return launch_exact_t<__half>(b, cells, ld, s64, s32, st);
    case CBX_BF16: return launch_exact_t<__nv_bfloat16>(b, cells, ld, s64, s32, st);
  }
  return fail(CBX_EINVAL, "unknown dtype");
}

}  // namespace cbx
