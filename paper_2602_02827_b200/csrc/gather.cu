// Candidate gather from an HBM-resident corpus (the fitted reranker's documents).
//
// The reference reranker stores its corpus once (ColBanditReranker.fit,
// colbandit/reranker.py:86-104) and scores a candidate pool per query
// (reranker.py:115-141). Here the corpus lives in HBM as a CSR token array;
// per call only query tokens and candidate ids cross PCIe. This kernel packs
// the candidates of every query into the contiguous CSR batch the scorer and
// the bandit consume: one exclusive scan of candidate lengths (single CTA,
// decoupled chunks) and a warp-per-document 16-byte vector copy.
#include "common.cuh"

namespace cbx {

constexpr int GA_SCAN_THREADS = 1024;
constexpr int GA_COPY_THREADS = 256;

// out_doc_off[j + 1] = sum of lengths of candidates 0..j; status[0] |= 1 on a bad id.
// One CTA; each thread scans 8 consecutive candidates serially, then a block scan of the totals.
constexpr int GA_PER = 8;
__global__ void __launch_bounds__(GA_SCAN_THREADS)
    gather_scan_kernel(const int64_t* __restrict__ corpus_off, int64_t n_corpus, const int64_t* __restrict__ cand,
                       int64_t n_cand, int64_t* __restrict__ out_off, int* __restrict__ status) {
  __shared__ int64_t warp_tot[GA_SCAN_THREADS / 32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry = 0;
    out_off[0] = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < n_cand; base += (int64_t)GA_SCAN_THREADS * GA_PER) {
    const int64_t j0 = base + (int64_t)tid * GA_PER;
    int64_t len[GA_PER];
    int64_t tot = 0;
#pragma unroll
    for (int u = 0; u < GA_PER; ++u) {
      len[u] = 0;
      const int64_t j = j0 + u;
      if (j < n_cand) {
        const int64_t id = cand[j];
        if (id < 0 || id >= n_corpus) atomicOr(status, 1);
        else len[u] = corpus_off[id + 1] - corpus_off[id];
      }
      tot += len[u];
    }
    int64_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < GA_SCAN_THREADS / 32 ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < GA_SCAN_THREADS / 32) warp_tot[lane] = w;
    }
    __syncthreads();
    int64_t run = x - tot + (warp ? warp_tot[warp - 1] : 0) + carry;  // exclusive prefix of this thread
#pragma unroll
    for (int u = 0; u < GA_PER; ++u) {
      run += len[u];
      if (j0 + u < n_cand) out_off[j0 + u + 1] = run;
    }
    __syncthreads();
    if (tid == GA_SCAN_THREADS - 1) carry = run;
    __syncthreads();
  }
}

// one warp per candidate: copy its token rows (16-byte vectors when rows allow, else 2-byte words; coalesced)
template <typename V>
__global__ void __launch_bounds__(GA_COPY_THREADS)
    gather_copy_kernel(const V* __restrict__ corpus, const int64_t* __restrict__ corpus_off,
                       const int64_t* __restrict__ cand, int64_t n_cand, const int64_t* __restrict__ out_off,
                       V* __restrict__ out, int64_t row_vecs, int64_t n_corpus) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (GA_COPY_THREADS / 32);
  for (int64_t j = (int64_t)blockIdx.x * (GA_COPY_THREADS / 32) + (threadIdx.x >> 5); j < n_cand; j += warps) {
    const int64_t id = cand[j];
    if (id < 0 || id >= n_corpus) continue;
    const V* src = corpus + corpus_off[id] * row_vecs;
    V* dst = out + out_off[j] * row_vecs;
    const int64_t n = (out_off[j + 1] - out_off[j]) * row_vecs;
    int64_t v = lane;
    for (; v + 96 < n; v += 128) {
      const V a = __ldg(src + v), b = __ldg(src + v + 32), c = __ldg(src + v + 64), d = __ldg(src + v + 96);
      dst[v] = a;
      dst[v + 32] = b;
      dst[v + 64] = c;
      dst[v + 96] = d;
    }
    for (; v < n; v += 32) dst[v] = __ldg(src + v);
  }
}

}  // namespace cbx

using namespace cbx;

extern "C" {

int cbx_gather_candidates(const void* corpus_tokens, const int64_t* corpus_doc_off, int64_t n_corpus_docs, int dim,
                          int dtype, const int64_t* cand_ids, int64_t n_cand, void* out_tokens, int64_t out_capacity,
                          int64_t* out_doc_off, int* status, void* stream) {
  if (n_cand <= 0) return CBX_OK;
  const size_t es = dtype_size(dtype);
  if (!es) return fail(CBX_EINVAL, "gather: unknown dtype");
  if (!corpus_tokens || !corpus_doc_off || !cand_ids || !out_tokens || !out_doc_off || !status)
    return fail(CBX_EINVAL, "gather: NULL buffer");
  (void)out_capacity;  // the caller sized out_tokens from host-side candidate lengths
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  gather_scan_kernel<<<1, GA_SCAN_THREADS, 0, st>>>(corpus_doc_off, n_corpus_docs, cand_ids, n_cand, out_doc_off,
                                                      status);
  CBX_LAUNCH_CHECK("gather_scan_kernel launch");
  const int grid = (int)std::min<int64_t>((n_cand + 7) / 8, (int64_t)sm_count() * 16);
  const bool vec16 = ((dim * es) % 16 == 0) &&
                     !((reinterpret_cast<uintptr_t>(corpus_tokens) | reinterpret_cast<uintptr_t>(out_tokens)) & 15);
  if (vec16)
    gather_copy_kernel<uint4><<<grid, GA_COPY_THREADS, 0, st>>>(
        static_cast<const uint4*>(corpus_tokens), corpus_doc_off, cand_ids, n_cand, out_doc_off,
        static_cast<uint4*>(out_tokens), (int64_t)dim * es / 16, n_corpus_docs);
  else
    gather_copy_kernel<uint16_t><<<grid, GA_COPY_THREADS, 0, st>>>(
        static_cast<const uint16_t*>(corpus_tokens), corpus_doc_off, cand_ids, n_cand, out_doc_off,
        static_cast<uint16_t*>(out_tokens), (int64_t)dim * es / 2, n_corpus_docs);
  CBX_LAUNCH_CHECK("gather_copy_kernel launch");
  return CBX_OK;
}

}  // extern "C"
