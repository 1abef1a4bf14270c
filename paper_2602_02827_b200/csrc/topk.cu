// Per-query Top-K by (-score, index) — replaces MaxSimOracle.exact_topk
// (colbandit/oracle.py:229-235: np.lexsort((arange(N), -scores))[:k], ties to
// the lower index) for every query of a batch in one stream-ordered call.
//
// Scores become 64-bit keys whose ascending order is descending score
// (-0.0 folded onto +0.0); the document index breaks ties. Each pass sorts
// segments of S keys with a shared-memory bitonic network (one CTA per
// (segment, query)) and keeps the first K; passes repeat until one segment per
// query remains. S <= 16384, K <= S / 2.
#include "common.cuh"

namespace cbx {

constexpr int TK_THREADS = 1024;
constexpr uint64_t TK_SENTINEL = ~0ull;

__device__ __forceinline__ float key_to_f32(uint64_t key) {
  uint32_t u = ~(uint32_t)key;
  uint32_t bits = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  return __uint_as_float(bits);
}
__device__ __forceinline__ double key_to_f64(uint64_t key) {
  uint64_t u = ~key;
  uint64_t bits = (u & 0x8000000000000000ull) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)bits);
}

template <typename ScoreT>
__device__ __forceinline__ uint64_t score_key(ScoreT s);
template <>
__device__ __forceinline__ uint64_t score_key<float>(float s) { return desc_key_f32(s); }
template <>
__device__ __forceinline__ uint64_t score_key<double>(double s) { return desc_key_f64(s); }

// FIRST: read raw scores (count per query from q_doc_off); else read (key, idx)
// pairs with a uniform per-query count. LAST: write decoded Top-K outputs.
template <typename ScoreT, bool FIRST, bool LAST>
__global__ void __launch_bounds__(TK_THREADS)
    topk_pass_kernel(const ScoreT* __restrict__ scores, const int64_t* __restrict__ q_doc_off,
                     const uint64_t* __restrict__ in_key, const uint32_t* __restrict__ in_idx, int64_t in_count,
                     uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_idx, int64_t out_cap, int S, int K,
                     int32_t* __restrict__ topk_idx, ScoreT* __restrict__ topk_val) {
  extern __shared__ __align__(16) uint8_t tk_smem[];
  uint64_t* key = reinterpret_cast<uint64_t*>(tk_smem);
  uint32_t* idx = reinterpret_cast<uint32_t*>(key + S);
  const int64_t q = blockIdx.y;
  const int64_t seg = blockIdx.x;
  int64_t n, base;
  if (FIRST) {
    base = q_doc_off[q];
    n = q_doc_off[q + 1] - base;
  } else {
    base = q * in_count;
    n = in_count;
  }
  const int64_t s0 = seg * (int64_t)S;
  for (int i = threadIdx.x; i < S; i += TK_THREADS) {
    const int64_t e = s0 + i;
    uint64_t k = TK_SENTINEL;
    uint32_t x = 0xFFFFFFFFu;
    if (e < n) {
      if (FIRST) {
        k = score_key<ScoreT>(scores[base + e]);
        x = (uint32_t)e;
      } else {
        k = in_key[base + e];
        x = in_idx[base + e];
      }
    }
    key[i] = k;
    idx[i] = x;
  }
  __syncthreads();
  for (int k = 2; k <= S; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < S; i += TK_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = key[i], b = key[ixj];
          const uint32_t ia = idx[i], ib = idx[ixj];
          const bool a_gt = (a > b) || (a == b && ia > ib);
          const bool up = (i & k) == 0;
          if (up == a_gt) {
            key[i] = b; key[ixj] = a;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < K; r += TK_THREADS) {
    if (LAST) {
      topk_idx[q * K + r] = (int32_t)idx[r];
      if (topk_val) {
        if constexpr (std::is_same<ScoreT, float>::value) topk_val[q * K + r] = key_to_f32(key[r]);
        else topk_val[q * K + r] = key_to_f64(key[r]);
      }
    } else {
      out_key[q * out_cap + seg * K + r] = key[r];
      out_idx[q * out_cap + seg * K + r] = idx[r];
    }
  }
}

static int seg_size(int64_t n, int K) {
  int64_t want = std::max<int64_t>(n, 2 * (int64_t)K);
  int S = 1024;
  while (S < want && S < 8192) S <<= 1;
  if (2 * K > S) S = 16384;
  return S;
}

size_t topk_workspace_bytes(int64_t n_queries, int64_t max_q_docs, int K) {
  if (K <= 0 || max_q_docs <= 0) return 0;
  int S = seg_size(max_q_docs, K);
  int64_t nseg = (max_q_docs + S - 1) / S;
  if (nseg <= 1) return 0;
  int64_t cap = nseg * K;
  return 2 * align_up((size_t)(n_queries * cap) * 12, 256);
}

template <typename ScoreT>
static int launch_topk_t(const ScoreT* scores, const int64_t* q_doc_off, int64_t nq, int64_t max_q_docs, int K,
                         int32_t* topk_idx, ScoreT* topk_val, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (K < 0) return fail(CBX_EINVAL, "k must be non-negative");
  if (K == 0 || nq == 0) return CBX_OK;
  if (K > 8192) return fail(CBX_EINVAL, "k > 8192 is not supported by the device Top-K");
  if (K > max_q_docs) return fail(CBX_EINVAL, "k exceeds the candidate pool");
  if (nq > 65535) return fail(CBX_EINVAL, "too many queries in one Top-K call (max 65535)");
  size_t need = topk_workspace_bytes(nq, max_q_docs, K);
  if (ws_bytes < need) return fail(CBX_EINVAL, "Top-K workspace too small");
  int S = seg_size(max_q_docs, K);
  int64_t nseg = (max_q_docs + S - 1) / S;
  size_t smem = (size_t)S * 12;
  auto k_first_last = topk_pass_kernel<ScoreT, true, true>;
  auto k_first = topk_pass_kernel<ScoreT, true, false>;
  auto k_mid = topk_pass_kernel<ScoreT, false, false>;
  auto k_last = topk_pass_kernel<ScoreT, false, true>;
  for (auto kf : {k_first_last, k_first, k_mid, k_last})
    CBX_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 12));
  if (nseg == 1) {
    k_first_last<<<dim3(1, (unsigned)nq), TK_THREADS, smem, st>>>(scores, q_doc_off, nullptr, nullptr, 0, nullptr,
                                                                   nullptr, 0, S, K, topk_idx, topk_val);
    CBX_LAUNCH_CHECK("topk_pass_kernel launch");
    return CBX_OK;
  }
  const size_t half = need / 2;
  uint64_t* key_a = static_cast<uint64_t*>(ws);
  uint32_t* idx_a = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + align_up(half * 8 / 12, 256));
  uint64_t* key_b = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ws) + half);
  uint32_t* idx_b = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + half + align_up(half * 8 / 12, 256));
  int64_t cap = nseg * K;
  k_first<<<dim3((unsigned)nseg, (unsigned)nq), TK_THREADS, smem, st>>>(scores, q_doc_off, nullptr, nullptr, 0, key_a,
                                                                         idx_a, cap, S, K, nullptr, nullptr);
  CBX_LAUNCH_CHECK("topk_pass_kernel launch");
  int64_t count = cap;
  bool in_a = true;
  while (true) {
    int S2 = seg_size(count, K);
    int64_t nseg2 = (count + S2 - 1) / S2;
    const uint64_t* ik = in_a ? key_a : key_b;
    const uint32_t* ii = in_a ? idx_a : idx_b;
    uint64_t* ok = in_a ? key_b : key_a;
    uint32_t* oi = in_a ? idx_b : idx_a;
    size_t smem2 = (size_t)S2 * 12;
    if (nseg2 == 1) {
      k_last<<<dim3(1, (unsigned)nq), TK_THREADS, smem2, st>>>(nullptr, nullptr, ik, ii, count, nullptr, nullptr, 0,
                                                               S2, K, topk_idx, topk_val);
      CBX_LAUNCH_CHECK("topk_pass_kernel launch");
      return CBX_OK;
    }
    int64_t cap2 = nseg2 * K;
    k_mid<<<dim3((unsigned)nseg2, (unsigned)nq), TK_THREADS, smem2, st>>>(nullptr, nullptr, ik, ii, count, ok, oi,
                                                                          cap2, S2, K, nullptr, nullptr);
    CBX_LAUNCH_CHECK("topk_pass_kernel launch");
    count = cap2;
    in_a = !in_a;
  }
}

int launch_topk_f32(const float* s, const int64_t* off, int64_t nq, int64_t mx, int K, int32_t* ti, float* tv,
                    void* ws, size_t wb, cudaStream_t st) {
  return launch_topk_t<float>(s, off, nq, mx, K, ti, tv, ws, wb, st);
}
int launch_topk_f64(const double* s, const int64_t* off, int64_t nq, int64_t mx, int K, int32_t* ti, double* tv,
                    void* ws, size_t wb, cudaStream_t st) {
  return launch_topk_t<double>(s, off, nq, mx, K, ti, tv, ws, wb, st);
}

}  // namespace cbx
