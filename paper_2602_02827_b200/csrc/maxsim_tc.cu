// K1 — dense MaxSim scorer on the 5th-generation tensor cores (sm_100a).
//
// Replaces the reference's per-document float64 GEMM + column max + fsum
// (colbandit/oracle.py:57-67 token_scores, 205-215 row_values, 222-227
// full_score) for a whole batch of queries at once.
//
// Orientation: the query is the MMA "A" operand (M = 128 rows, of which the
// first Lq are real query tokens), a tile of TILE_N consecutive document
// tokens is "B" (N = TILE_N), K = embedding dim. The fp32 accumulator lives in
// TMEM as 128 lanes x TILE_N columns: lane t holds <q_t, e_j> for the tile's
// doc tokens j. The epilogue thread for lane t therefore owns one query token
// and computes the per-document max along its own columns — no cross-lane
// shuffles for the max; one butterfly sum per finished document gives
// S_d = sum_t max_j <q_t, e_j>. No score matrix ever reaches HBM.
//
// Work unit = "chunk": the documents of one query whose first token falls in
// a fixed window of T tokens. A chunk is processed start-to-end by one CTA,
// so a document that spans tiles carries its running max in registers.
//
// Warp roles (256 threads, one CTA per SM, persistent over chunks):
//   warp 0      TMA producer: query tile (2 slots) + doc tiles (NS-stage ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4..7  epilogue: tcgen05.ld -> segmented max -> sum -> scores
// Pipelines: smem full/empty (TMA <-> MMA), query full/empty, TMEM
// accumulator full/empty (MMA <-> epilogue, 4 x TILE_N columns).
#include <cuda.h>

#include "common.cuh"
#include "ptx.cuh"

namespace cbx {

constexpr int TC_THREADS = 256;
constexpr int TC_EPI_WARP0 = 4;
constexpr int TC_ACC_BUFS = 4;
constexpr int TC_MAX_TILE_N = 128;
constexpr int TC_MAX_STAGES = 8;

struct TcParams {
  const int64_t* q_tok_off;
  const int64_t* d_tok_off;
  const int64_t* q_doc_off;
  float* scores;
  int64_t n_chunks;      // n_queries * chunks_per_query
  int64_t chunks_per_query;
  int64_t chunk_tokens;  // T
  uint32_t idesc;
  int32_t tile_n;
  int32_t kblocks;       // ceil(dim / 64)
  int32_t lqp;           // query rows staged per slot (max Lq rounded up to 8)
  int32_t stages;
  int32_t clamp_negative;
  uint32_t q_slot_bytes;
  uint32_t stage_bytes;
};

struct ChunkInfo {
  int64_t doc0, doc1;   // global doc range [doc0, doc1)
  int64_t cs, ce;       // token range [cs, ce)
  int64_t q_tok0;       // first query token row
  int32_t lq;
  int32_t ntiles;
};

// first doc index in [lo, hi) whose start offset is >= x
__device__ __forceinline__ int64_t lower_bound_start(const int64_t* __restrict__ d_tok_off, int64_t lo, int64_t hi,
                                                     int64_t x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(d_tok_off + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool decode_chunk(const TcParams& p, int64_t g, ChunkInfo& c) {
  int64_t q = g / p.chunks_per_query;
  int64_t k = g - q * p.chunks_per_query;
  int64_t db = __ldg(p.q_doc_off + q), de = __ldg(p.q_doc_off + q + 1);
  if (db >= de) return false;
  int64_t qs = __ldg(p.d_tok_off + db);
  int64_t x0 = qs + k * p.chunk_tokens, x1 = x0 + p.chunk_tokens;
  c.doc0 = lower_bound_start(p.d_tok_off, db, de, x0);
  c.doc1 = lower_bound_start(p.d_tok_off, c.doc0, de, x1);
  if (c.doc0 >= c.doc1) return false;
  c.cs = __ldg(p.d_tok_off + c.doc0);
  c.ce = __ldg(p.d_tok_off + c.doc1);
  c.q_tok0 = __ldg(p.q_tok_off + q);
  c.lq = (int32_t)(__ldg(p.q_tok_off + q + 1) - c.q_tok0);
  c.ntiles = (int32_t)((c.ce - c.cs + p.tile_n - 1) / p.tile_n);
  return true;
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    maxsim_tc_kernel(const __grid_constant__ CUtensorMap tmap_d, const __grid_constant__ CUtensorMap tmap_q,
                     const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_slots = smem;                                   // 2 x q_slot_bytes
  uint8_t* stages = smem + 2 * p.q_slot_bytes;               // stages x stage_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)p.stages * p.stage_bytes);
  uint64_t* full = bars;                                     // [stages]
  uint64_t* empty = bars + TC_MAX_STAGES;                    // [stages]
  uint64_t* qfull = bars + 2 * TC_MAX_STAGES;                // [2]
  uint64_t* qempty = qfull + 2;                              // [2]
  uint64_t* tfull = qempty + 2;                              // [4]
  uint64_t* tempty = tfull + TC_ACC_BUFS;                    // [4]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + TC_ACC_BUFS);
  float* part = reinterpret_cast<float*>(bars + 64);         // [2][4][TC_MAX_TILE_N]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&qfull[s], 1);
      ptx::mbar_init(&qempty[s], 1);
    }
    for (int s = 0; s < TC_ACC_BUFS; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_d);
    ptx::prefetch_tmap(&tmap_q);
  }
  if (warp == 1) ptx::tmem_alloc<TC_ACC_BUFS * TC_MAX_TILE_N>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, qs = 0, qphase = 0;
      const uint64_t pol = ptx::policy_evict_first();
      for (int64_t g = blockIdx.x; g < p.n_chunks; g += gridDim.x) {
        ChunkInfo c;
        if (!decode_chunk(p, g, c)) continue;
        ptx::mbar_wait(&qempty[qs], qphase ^ 1);
        ptx::mbar_arrive_expect_tx(&qfull[qs], p.q_slot_bytes);
        for (int kb = 0; kb < p.kblocks; ++kb)
          ptx::tma_load_2d(q_slots + qs * p.q_slot_bytes + kb * p.lqp * 128, &tmap_q, &qfull[qs], kb * 64,
                           (int32_t)c.q_tok0);
        if (++qs == 2) { qs = 0; qphase ^= 1; }
        for (int t = 0; t < c.ntiles; ++t) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], p.stage_bytes);
          const int32_t row = (int32_t)(c.cs + (int64_t)t * p.tile_n);
          uint8_t* dst = stages + (size_t)stage * p.stage_bytes;
          for (int kb = 0; kb < p.kblocks; ++kb)
            ptx::tma_load_2d_hint(dst + kb * p.tile_n * 128, &tmap_d, &full[stage], kb * 64, row, pol);
          if (++stage == (uint32_t)p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, qs = 0, qphase = 0, acc = 0, aphase = 0;
      for (int64_t g = blockIdx.x; g < p.n_chunks; g += gridDim.x) {
        ChunkInfo c;
        if (!decode_chunk(p, g, c)) continue;
        ptx::mbar_wait(&qfull[qs], qphase);
        ptx::tc_fence_after();
        const uint32_t q_addr = ptx::smem_u32(q_slots + qs * p.q_slot_bytes);
        for (int t = 0; t < c.ntiles; ++t) {
          ptx::mbar_wait(&tempty[acc], aphase ^ 1);
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t b_addr = ptx::smem_u32(stages + (size_t)stage * p.stage_bytes);
          const uint32_t d_tmem = tmem_base + acc * TC_MAX_TILE_N;
          for (int kb = 0; kb < p.kblocks; ++kb) {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              uint64_t ad = ptx::smem_desc_sw128(q_addr + kb * p.lqp * 128 + k4 * 32);
              uint64_t bd = ptx::smem_desc_sw128(b_addr + kb * p.tile_n * 128 + k4 * 32);
              ptx::tc_mma_f16(d_tmem, ad, bd, p.idesc, (kb | k4) != 0);
            }
          }
          ptx::tc_commit(&empty[stage]);
          ptx::tc_commit(&tfull[acc]);
          if (++stage == (uint32_t)p.stages) { stage = 0; phase ^= 1; }
          if (++acc == TC_ACC_BUFS) { acc = 0; aphase ^= 1; }
        }
        ptx::tc_commit(&qempty[qs]);
        if (++qs == 2) { qs = 0; qphase ^= 1; }
      }
    }
  } else if (warp >= TC_EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - TC_EPI_WARP0;  // TMEM lane quadrant
    uint32_t acc = 0, aphase = 0, tile_parity = 0;
    const float init = p.clamp_negative ? 0.0f : -INFINITY;
    for (int64_t g = blockIdx.x; g < p.n_chunks; g += gridDim.x) {
      ChunkInfo c;
      if (!decode_chunk(p, g, c)) continue;
      const int nact = (c.lq + 31) >> 5;
      const bool active = ew < nact;
      const bool lane_valid = ew * 32 + lane < c.lq;
      float cur = init;
      // window of 32 document end offsets, one per lane
      int64_t win = c.doc0;
      int64_t ends = (win + lane < c.doc1) ? __ldg(p.d_tok_off + win + 1 + lane) : INT64_MAX;
      int64_t doc = c.doc0;
      int64_t doc_end = __shfl_sync(0xffffffffu, ends, 0);
      for (int t = 0; t < c.ntiles; ++t) {
        ptx::mbar_wait(&tfull[acc], aphase);
        ptx::tc_fence_after();
        const int64_t tbase = c.cs + (int64_t)t * p.tile_n;
        const int ncols = (int)(c.ce - tbase < p.tile_n ? c.ce - tbase : p.tile_n);
        float v[TC_MAX_TILE_N / 32][32];
        if (active) {
          const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * TC_MAX_TILE_N;
#pragma unroll
          for (int b = 0; b < TC_MAX_TILE_N / 32; ++b)
            if (b * 32 < ncols) ptx::tmem_ld_32x32b_x32(taddr + b * 32, v[b]);
          ptx::tmem_ld_wait();
        }
        ptx::tc_fence_before();
        if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        if (++acc == TC_ACC_BUFS) { acc = 0; aphase ^= 1; }
        if (!active) continue;

        int nfin = 0;
        int64_t fin0 = doc;
        float* mypart = part + (tile_parity * 4 + ew) * TC_MAX_TILE_N;
#pragma unroll
        for (int b = 0; b < TC_MAX_TILE_N / 32; ++b) {
          if (b * 32 >= ncols) break;
          const int nc = min(32, ncols - b * 32);
          const int64_t g0 = tbase + b * 32;
          int s = 0;
          while (true) {
            const int64_t end_rel = doc_end - g0;
            const int e = (int)(end_rel < nc ? end_rel : nc);
            float m = cur;
            if (s == 0 && e == 32) {
              float a[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) a[j] = fmaxf(v[b][j], v[b][j + 16]);
#pragma unroll
              for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                for (int j = 0; j < w; ++j) a[j] = fmaxf(a[j], a[j + w]);
              m = fmaxf(m, a[0]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j >= s && j < e) m = fmaxf(m, v[b][j]);
            }
            cur = m;
            if (end_rel > nc) break;  // document continues past this block
            // document `doc` ends inside this block: finalize it
            float x = warp_sum(lane_valid ? cur : 0.0f);
            if (nact == 1) {
              if (lane == 0) p.scores[doc] = x;
            } else {
              if (lane == 0) mypart[nfin] = x;
            }
            ++nfin;
            cur = init;
            ++doc;
            if (doc - win == 32) {
              win = doc;
              ends = (win + lane < c.doc1) ? __ldg(p.d_tok_off + win + 1 + lane) : INT64_MAX;
            }
            doc_end = __shfl_sync(0xffffffffu, ends, (int)(doc - win));
            s = e;
            if (s >= nc) break;
          }
        }
        if (nact > 1) {
          // combine per-quadrant partial sums in a fixed order
          asm volatile("bar.sync 1, %0;" ::"r"(nact * 32) : "memory");
          if (ew == 0) {
            const float* pp = part + tile_parity * 4 * TC_MAX_TILE_N;
            for (int j = lane; j < nfin; j += 32) {
              float sacc = pp[j];
              for (int w = 1; w < nact; ++w) sacc += pp[w * TC_MAX_TILE_N + j];
              p.scores[fin0 + j] = sacc;
            }
          }
          tile_parity ^= 1;
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TC_ACC_BUFS * TC_MAX_TILE_N>(tmem_base);
  }
}

// ----------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static int make_tmap(CUtensorMap* m, const void* base, int dtype, int64_t rows, int32_t dim, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(CBX_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)dim, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)dim * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dtype == CBX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CBX_ECUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return CBX_OK;
}

bool tc_supported(const cbx_batch* b) {
  return (b->dtype == CBX_F16 || b->dtype == CBX_BF16) && b->max_lq >= 1 && b->max_lq <= 128 && b->dim % 8 == 0 &&
         b->dim <= 512 && b->n_d_tokens < (int64_t(1) << 31) && b->n_q_tokens < (int64_t(1) << 31);
}

int launch_maxsim_tc(const cbx_batch* b, float* scores, cudaStream_t stream) {
  if (!tc_supported(b)) return fail(CBX_EINVAL, "tcgen05 scorer needs f16/bf16 tokens, Lq <= 128, dim % 8 == 0");
  if (b->n_docs == 0 || b->n_queries == 0) return CBX_OK;
  const int kblocks = (b->dim + 63) / 64;
  const int tile_n = kblocks <= 2 ? 128 : 64;
  const int lqp = (b->max_lq + 7) / 8 * 8;
  const uint32_t q_slot_bytes = (uint32_t)(kblocks * lqp * 128);
  const uint32_t stage_bytes = (uint32_t)(kblocks * tile_n * 128);
  const size_t bar_bytes = 512 + 2 * 4 * TC_MAX_TILE_N * sizeof(float);  // barriers + partial sums
  const size_t budget = 227 * 1024 - 1024 /*align slack*/ - bar_bytes - 2 * q_slot_bytes;
  int stages = (int)std::min<size_t>(TC_MAX_STAGES, budget / stage_bytes);
  if (stages < 2) return fail(CBX_EINVAL, "tcgen05 scorer: query tile too large for shared memory");
  // the A operand always spans 128 rows; rows past Lq read (ignored) bytes that must lie inside the allocation
  const size_t smem = 1024 + 2 * (size_t)q_slot_bytes + (size_t)stages * stage_bytes + bar_bytes;
  if ((size_t)q_slot_bytes + (size_t)(kblocks - 1) * lqp * 128 + 128 * 128 >
      2 * (size_t)q_slot_bytes + (size_t)stages * stage_bytes)
    return fail(CBX_EINTERNAL, "tcgen05 scorer: shared layout too small for the 128-row A operand");

  CUtensorMap tmd, tmq;
  int rc = make_tmap(&tmd, b->d_tokens, b->dtype, b->n_d_tokens, b->dim, (uint32_t)tile_n);
  if (rc) return rc;
  rc = make_tmap(&tmq, b->q_tokens, b->dtype, b->n_q_tokens, b->dim, (uint32_t)lqp);
  if (rc) return rc;

  const int nsm = sm_count();
  TcParams p;
  p.q_tok_off = b->q_tok_off;
  p.d_tok_off = b->d_tok_off;
  p.q_doc_off = b->q_doc_off;
  p.scores = scores;
  // chunk window: enough chunks for ~6 per SM, never below 4 tiles or above 32k tokens
  int64_t total = std::max<int64_t>(b->n_d_tokens, 1);
  int64_t T = total / ((int64_t)nsm * 6);
  T = std::max<int64_t>(T, 4 * tile_n);
  T = std::min<int64_t>(T, 32768);
  T = (T + tile_n - 1) / tile_n * tile_n;
  p.chunk_tokens = T;
  p.chunks_per_query = std::max<int64_t>(1, (b->max_q_doc_tokens + T - 1) / T);
  p.n_chunks = p.chunks_per_query * b->n_queries;
  p.idesc = ptx::idesc_f16(b->dtype == CBX_BF16, 128, (uint32_t)tile_n);
  p.tile_n = tile_n;
  p.kblocks = kblocks;
  p.lqp = lqp;
  p.stages = stages;
  p.clamp_negative = b->clamp_negative;
  p.q_slot_bytes = q_slot_bytes;
  p.stage_bytes = stage_bytes;

  CBX_CUDA_CHECK(cudaFuncSetAttribute(maxsim_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = (int)std::min<int64_t>(p.n_chunks, nsm);
  maxsim_tc_kernel<<<grid, TC_THREADS, smem, stream>>>(tmd, tmq, p);
  CBX_LAUNCH_CHECK("maxsim_tc_kernel launch");
  return CBX_OK;
}

}  // namespace cbx
