// Stage-1 candidate scan — replaces colbandit/pipeline.py:105-158 (generate_candidates).
//
// For every query-token row r and the whole corpus (T token rows), the k'
// corpus tokens of highest similarity, ranked by (-similarity, global token
// index) exactly like np.lexsort((arange(T), -scores[:, t]))[:k'] on the
// reference's float64 scores (pipeline.py:137), similarity floored at 0 under
// clamp_negative (oracle.py:65-66). Two device paths, identical results:
//
// * SIMT (any dtype): the corpus is cut into chunks; a CUDA-core kernel writes
//   float64 similarities of a chunk (same fma order as the exact cell kernel,
//   so a neighbour's value equals the cell the oracle later reveals), the
//   segmented bitonic Top-K keeps k' per row and chunk, a last Top-K merges
//   the chunk winners (chunk order = token order, so ties stay lowest-index).
//
// * TC (fp16/bf16, large corpora): one persistent TMA + tcgen05 scan streams
//   the corpus once per 128 query rows (query rows = the MMA's M, 128 corpus
//   tokens = N, fp32 accumulators in TMEM). The epilogue keeps, per row, a
//   running k'-th best value theta (sorted top-k' in shared memory) and
//   appends every token with fp32 value >= theta - 2*eps_r to a per-(item,
//   row) list; eps_r = dim * 2^-19 * |q_r| * max_j |e_j| bounds the fp32
//   accumulation error (products of 16-bit inputs are exact). theta starts
//   from a pre-pass over every stride-th tile (the k'-th best of a corpus
//   sample is a lower bound on the global k'-th value), so the main scan
//   appends and inserts almost only true contenders. A refine kernel
//   per row takes T_f = the k'-th best fp32 value over all items, recomputes
//   every listed token with fp32 >= T_f - 2*eps_r in float64 and sorts them by
//   (-value, index). Every true Top-k' token has fp32 >= T_f - 2*eps_r, so the
//   result is exact. Overflowing a list, or a k'-th value of exactly 0 under
//   clamping (zero ties resolved by corpus order), sets status: the caller
//   re-runs the SIMT path.
#include <cuda.h>

#include "common.cuh"
#include "ptx.cuh"

namespace cbx {

int make_tmap(CUtensorMap* m, const void* base, int dtype, int64_t rows, int32_t dim, uint32_t box_rows);
size_t topk_workspace_bytes(int64_t n_queries, int64_t max_q_docs, int K);
int launch_topk_f64(const double* s, const int64_t* off, int64_t nq, int64_t mx, int K, int32_t* ti, double* tv,
                    void* ws, size_t wb, cudaStream_t st);

template <typename T>
using S1Store = typename std::conditional<std::is_same<T, double>::value, double, float>::type;

// ============================================================ SIMT path
constexpr int SX_ROWS = 64, SX_TOKS = 64, SX_THREADS = 256;

// sims[r * C + j] = <e_{c0+j}, q_r> (float64, clamped), -inf for j >= cn (chunk padding)
template <typename T>
__global__ void __launch_bounds__(SX_THREADS)
    stage1_sims_kernel(const T* __restrict__ q, int64_t R, const T* __restrict__ d, int64_t c0, int64_t cn,
                       int64_t C, int dim, int clamp, double* __restrict__ sims) {
  using S = S1Store<T>;
  extern __shared__ __align__(16) uint8_t sx_smem[];
  const int dp = dim + 1;
  S* qs = reinterpret_cast<S*>(sx_smem);
  S* ts = qs + SX_ROWS * dp;
  const int64_t r0 = (int64_t)blockIdx.y * SX_ROWS, j0 = (int64_t)blockIdx.x * SX_TOKS;
  for (int i = threadIdx.x; i < SX_ROWS * dim; i += SX_THREADS) {
    const int r = i / dim, k = i - r * dim;
    qs[r * dp + k] = r0 + r < R ? (S)Elem<T>::to_d(q[(r0 + r) * dim + k]) : (S)0;
    ts[r * dp + k] = j0 + r < cn ? (S)Elem<T>::to_d(d[(c0 + j0 + r) * dim + k]) : (S)0;
  }
  __syncthreads();
  const int j = threadIdx.x & (SX_TOKS - 1), rg = threadIdx.x / SX_TOKS;  // rows rg + 4 i
  double acc[SX_ROWS / 4];
#pragma unroll
  for (int i = 0; i < SX_ROWS / 4; ++i) acc[i] = 0.0;
  for (int k = 0; k < dim; ++k) {
    const double e = (double)ts[j * dp + k];
#pragma unroll
    for (int i = 0; i < SX_ROWS / 4; ++i) acc[i] = fma(e, (double)qs[(rg + 4 * i) * dp + k], acc[i]);
  }
#pragma unroll
  for (int i = 0; i < SX_ROWS / 4; ++i) {
    const int64_t r = r0 + rg + 4 * i;
    if (r >= R) break;
    double v = acc[i];
    if (clamp) v = v > 0.0 ? v : 0.0;
    sims[r * C + j0 + j] = j0 + j < cn ? v : -INFINITY;
  }
}

__global__ void stage1_offsets_kernel(int64_t* off, int64_t n, int64_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    off[i] = i * stride;
}

// chunk winners -> candidate list [r][chunk * kp + i] (value, global token index)
__global__ void stage1_scatter_kernel(const int32_t* __restrict__ idx, const double* __restrict__ val, int64_t R,
                                      int kp, int64_t chunk, int64_t nch, int64_t c0, double* __restrict__ cv,
                                      int64_t* __restrict__ ct) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R * kp; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / kp, s = i - r * kp;
    cv[r * nch * kp + chunk * kp + s] = val[i];
    ct[r * nch * kp + chunk * kp + s] = c0 + idx[i];
  }
}

__global__ void stage1_final_kernel(const int32_t* __restrict__ pos, const double* __restrict__ val,
                                    const int64_t* __restrict__ ct, int64_t R, int kp, int64_t width,
                                    int64_t* __restrict__ nb_tok, double* __restrict__ nb_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R * kp; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / kp;
    nb_tok[i] = ct[r * width + pos[i]];
    nb_val[i] = val[i];
  }
}

struct SxPlan {
  int64_t C, nch;
  size_t o_sims, o_off1, o_off2, o_idx, o_val, o_cv, o_ct, o_pos, o_fval, o_tk, total;
};

static SxPlan plan_simt(int64_t R, int64_t T, int kp) {
  SxPlan p;
  int64_t C = std::max<int64_t>(4096, ((int64_t)1 << 25) / std::max<int64_t>(R, 1));
  C = std::max<int64_t>(C, 2 * (int64_t)kp);
  C = std::min<int64_t>(C, (T + SX_TOKS - 1) / SX_TOKS * SX_TOKS);
  C = std::max<int64_t>(C, (int64_t)kp);
  C = (C + SX_TOKS - 1) / SX_TOKS * SX_TOKS;
  p.C = C;
  p.nch = (T + C - 1) / C;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  p.o_sims = take(8 * (size_t)R * C);
  p.o_off1 = take(8 * (size_t)(R + 1));
  p.o_off2 = take(8 * (size_t)(R + 1));
  p.o_idx = take(4 * (size_t)R * kp);
  p.o_val = take(8 * (size_t)R * kp);
  p.o_cv = take(8 * (size_t)R * p.nch * kp);
  p.o_ct = take(8 * (size_t)R * p.nch * kp);
  p.o_pos = take(4 * (size_t)R * kp);
  p.o_fval = take(8 * (size_t)R * kp);
  p.o_tk = take(std::max(topk_workspace_bytes(R, C, kp), topk_workspace_bytes(R, p.nch * kp, kp)));
  p.total = o;
  return p;
}

template <typename T>
static int run_simt(const cbx_batch* b, int kp, int64_t* nb_tok, double* nb_val, uint8_t* ws, cudaStream_t st) {
  using S = S1Store<T>;
  const int64_t R = b->n_q_tokens, Tn = b->n_d_tokens;
  SxPlan p = plan_simt(R, Tn, kp);
  double* sims = reinterpret_cast<double*>(ws + p.o_sims);
  int64_t* off1 = reinterpret_cast<int64_t*>(ws + p.o_off1);
  int64_t* off2 = reinterpret_cast<int64_t*>(ws + p.o_off2);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + p.o_idx);
  double* val = reinterpret_cast<double*>(ws + p.o_val);
  double* cv = reinterpret_cast<double*>(ws + p.o_cv);
  int64_t* ct = reinterpret_cast<int64_t*>(ws + p.o_ct);
  int32_t* pos = reinterpret_cast<int32_t*>(ws + p.o_pos);
  double* fval = reinterpret_cast<double*>(ws + p.o_fval);
  void* tk = ws + p.o_tk;
  const size_t tk_bytes = p.total - p.o_tk;
  const size_t smem = 2 * sizeof(S) * SX_ROWS * (b->dim + 1);
  if (smem > 227 * 1024) return fail(CBX_EINVAL, "stage-1 SIMT scan: embedding dim too large");
  CBX_CUDA_CHECK(cudaFuncSetAttribute(stage1_sims_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  stage1_offsets_kernel<<<64, 256, 0, st>>>(off1, R, p.C);
  stage1_offsets_kernel<<<64, 256, 0, st>>>(off2, R, p.nch * kp);
  CBX_LAUNCH_CHECK("stage1_offsets_kernel launch");
  const int sgrid = (int)std::min<int64_t>((R * kp + 255) / 256, 4096);
  for (int64_t c = 0; c < p.nch; ++c) {
    const int64_t c0 = c * p.C, cn = std::min<int64_t>(p.C, Tn - c0);
    dim3 grid((unsigned)(p.C / SX_TOKS), (unsigned)((R + SX_ROWS - 1) / SX_ROWS));
    stage1_sims_kernel<T><<<grid, SX_THREADS, smem, st>>>(static_cast<const T*>(b->q_tokens), R,
                                                           static_cast<const T*>(b->d_tokens), c0, cn, p.C, b->dim,
                                                           b->clamp_negative, sims);
    CBX_LAUNCH_CHECK("stage1_sims_kernel launch");
    if (p.nch == 1) {  // one chunk: its winners are the answer (chunk positions == token indices)
      int rc = launch_topk_f64(sims, off1, R, p.C, kp, idx, val, tk, tk_bytes, st);
      if (rc) return rc;
      stage1_scatter_kernel<<<sgrid, 256, 0, st>>>(idx, val, R, kp, 0, 1, 0, nb_val, nb_tok);
      CBX_LAUNCH_CHECK("stage1_scatter_kernel launch");
      return CBX_OK;
    }
    int rc = launch_topk_f64(sims, off1, R, p.C, kp, idx, val, tk, tk_bytes, st);
    if (rc) return rc;
    stage1_scatter_kernel<<<sgrid, 256, 0, st>>>(idx, val, R, kp, c, p.nch, c0, cv, ct);
    CBX_LAUNCH_CHECK("stage1_scatter_kernel launch");
  }
  int rc = launch_topk_f64(cv, off2, R, p.nch * kp, kp, pos, fval, tk, tk_bytes, st);
  if (rc) return rc;
  stage1_final_kernel<<<sgrid, 256, 0, st>>>(pos, fval, ct, R, kp, p.nch * kp, nb_tok, nb_val);
  CBX_LAUNCH_CHECK("stage1_final_kernel launch");
  return CBX_OK;
}

// ============================================================ TC path
constexpr int S1_THREADS = 256;
constexpr int S1_EPI_WARP0 = 4;
constexpr int S1_ACC = 4;
constexpr int S1_TILE = 128;
constexpr int S1_MAX_STAGES = 6;
constexpr int S1_MAX_KP = 256;  // per-row sorted tops live in shared memory (4 B x 128 rows x k')
constexpr int S1_FCAP = 2048;  // refined candidates per row
constexpr int S1_MIN_TOKENS = 8192;

struct S1Params {
  int64_t R, T;
  int32_t RB, P, NT, kp, cap, kblocks, stages;  // cap: list entries per (item, row)
  int32_t sample;   // 1: threshold pre-pass over every stride-th tile (tile maxima only)
  int32_t stride;   // tile stride of the visited sequence
  int32_t NS;       // tiles in the visited sequence
  int32_t tile_n;                               // corpus tokens per MMA tile (N): 128, or 64 for d > 128 when needed
  uint32_t idesc, q_slot_bytes, stage_bytes;
  const float* eps;
  unsigned int* gthr;  // [R] order-preserving keys of the best published k'-th value per row
  int32_t* cnt;   // [items][128]
  uint2* ent;     // [items][128][cap]: (fp32 bits, token)
  float* topv;    // [items][128][kp] descending, -inf padded
  float* tmax;    // pre-pass: [NS][R] tile maxima
  int* status;
};

__global__ void stage1_eps_kernel(const void* q, int dtype, int64_t R, int dim, float norm_max, float* eps) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= R) return;
  double s = 0.0;
  for (int k = lane; k < dim; k += 32) {
    double x = dtype == CBX_BF16 ? (double)__bfloat162float(static_cast<const __nv_bfloat16*>(q)[r * dim + k])
                                 : (double)__half2float(static_cast<const __half*>(q)[r * dim + k]);
    s += x * x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) eps[r] = (float)((double)dim * 0x1p-19 * sqrt(s) * (double)norm_max * 1.0001 + 1e-30);
}

// order-preserving float <-> uint keys (atomicMax on floats of any sign)
__device__ __forceinline__ unsigned int ord_key(float x) {
  const unsigned int u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_val(unsigned int k) {
  if (k == 0u) return -INFINITY;  // nothing published yet
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__device__ __forceinline__ float s1_fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// max of 32 register values as a 3-input tree (depth 4)
__device__ __forceinline__ float s1_tree_max32(const float (&v)[32]) {
  float a[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) a[i] = s1_fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  a[10] = fmaxf(v[30], v[31]);
  const float b0 = s1_fmax3(a[0], a[1], a[2]), b1 = s1_fmax3(a[3], a[4], a[5]), b2 = s1_fmax3(a[6], a[7], a[8]);
  return s1_fmax3(s1_fmax3(b0, b1, b2), a[9], a[10]);
}

__global__ void __launch_bounds__(S1_THREADS, 1)
    stage1_scan_kernel(const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_q,
                       S1Params p) {
  extern __shared__ __align__(1024) uint8_t s1_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s1_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_slot = smem;
  uint8_t* stages = smem + p.q_slot_bytes;
  float* tops = reinterpret_cast<float*>(stages + (size_t)p.stages * p.stage_bytes);  // [kp][128]
  float* scratch = tops + (size_t)p.kp * 128;                                          // [32][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(scratch + 32 * 128);
  uint64_t* full = bars;
  uint64_t* empty = bars + S1_MAX_STAGES;
  uint64_t* qfull = bars + 2 * S1_MAX_STAGES;
  uint64_t* qempty = qfull + 1;
  uint64_t* tfull = qempty + 1;
  uint64_t* tempty = tfull + S1_ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + S1_ACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = p.RB * p.P;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(qfull, 1);
    ptx::mbar_init(qempty, 1);
    for (int s = 0; s < S1_ACC; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_d);
    ptx::prefetch_tmap(&tm_q);
  }
  if (warp == 1) ptx::tmem_alloc<S1_ACC * S1_TILE>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      uint32_t tg = 0, qphase = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int rb = item / p.P, pp = item - rb * p.P;
        const int t0 = (int)((int64_t)p.NS * pp / p.P), t1 = (int)((int64_t)p.NS * (pp + 1) / p.P);
        ptx::mbar_wait(qempty, qphase ^ 1);
        qphase ^= 1;
        ptx::mbar_arrive_expect_tx(qfull, (uint32_t)(p.kblocks * 16384));
        for (int kb = 0; kb < p.kblocks; ++kb) ptx::tma_load_2d(q_slot + kb * 16384, &tm_q, qfull, kb * 64, rb * 128);
        for (int t = t0; t < t1; ++t, ++tg) {
          const uint32_t stage = tg % (uint32_t)p.stages, ph = (tg / (uint32_t)p.stages) & 1u;
          ptx::mbar_wait(&empty[stage], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], p.stage_bytes);
          uint8_t* dst = stages + (size_t)stage * p.stage_bytes;
          for (int kb = 0; kb < p.kblocks; ++kb)
            ptx::tma_load_2d_hint(dst + kb * p.tile_n * 128, &tm_d, &full[stage], kb * 64, t * p.stride * p.tile_n,
                                  pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t tg = 0, qphase = 0, stage = 0, phase = 0;
      const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(q_slot));
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int rb = item / p.P, pp = item - rb * p.P;
        const int t0 = (int)((int64_t)p.NS * pp / p.P), t1 = (int)((int64_t)p.NS * (pp + 1) / p.P);
        ptx::mbar_wait(qfull, qphase);
        qphase ^= 1;
        ptx::tc_fence_after();
        for (int t = t0; t < t1; ++t, ++tg) {
          const uint32_t acc = tg & (S1_ACC - 1);
          ptx::mbar_wait(&tempty[acc], ((tg >> 2) & 1) ^ 1);
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(stages + (size_t)stage * p.stage_bytes));
          const uint32_t d_tmem = tmem_base + acc * S1_TILE;
          const uint32_t bstep = (uint32_t)(p.tile_n * 128) >> 4;
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            if (kb >= p.kblocks) break;
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              ptx::tc_mma_f16(d_tmem, ad0 + (uint64_t)(kb * 1024 + k4 * 2), bd0 + (uint64_t)(kb * bstep + k4 * 2),
                              p.idesc, (kb | k4) != 0);
          }
          ptx::tc_commit(&empty[stage]);
          ptx::tc_commit(&tfull[acc]);
          if (++stage == (uint32_t)p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::tc_commit(qempty);
      }
    }
  } else if (warp >= S1_EPI_WARP0) {
    const int quad = warp - S1_EPI_WARP0;
    const int rl = quad * 32 + lane;  // row within the 128-row block == TMEM lane
    const uint32_t tmem_lane = (uint32_t)(quad * 32) << 16;
    uint32_t tg = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int rb = item / p.P, pp = item - rb * p.P;
      const int t0 = (int)((int64_t)p.NS * pp / p.P), t1 = (int)((int64_t)p.NS * (pp + 1) / p.P);
      const int64_t r = (int64_t)rb * 128 + rl;
      const bool valid = r < p.R;
      const float eps2 = valid ? 2.0f * __ldg(p.eps + r) : 0.0f;
      const bool any_valid = (int64_t)rb * 128 + quad * 32 < p.R;  // warp-uniform: this quadrant holds rows
      // theta: k'-th best fp32 value of this item's row so far (sorted tops); gtheta: the pre-pass's k'-th
      // best over a strided sample of the corpus. Both are <= the global k'-th fp32 value, so
      // thr = max(theta, gtheta) - 2 eps never drops a token the refine needs.
      const float gtheta = (!p.sample && valid) ? ord_val(__ldg(p.gthr + r)) : -INFINITY;
      float theta = -INFINITY, thr = gtheta - eps2;
      int ntop = 0, cnt = 0;
      bool ovf = false;
      uint2* mylist = p.ent + ((size_t)item * 128 + rl) * p.cap;
      for (int t = t0; t < t1; ++t, ++tg) {
        const uint32_t acc = tg & (S1_ACC - 1);
        ptx::mbar_wait(&tfull[acc], (tg >> 2) & 1);
        ptx::tc_fence_after();
        float v[4][32];
        const uint32_t taddr = tmem_base + tmem_lane + acc * S1_TILE;
        if (any_valid) {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (b * 32 < p.tile_n) ptx::tmem_ld_32x32b_x32(taddr + b * 32, v[b]);
          ptx::tmem_ld_wait();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        if (!any_valid) continue;
        const int64_t tb = (int64_t)t * p.stride * p.tile_n;
        const int ncols = p.T - tb < p.tile_n ? (int)(p.T - tb) : p.tile_n;
        if (ncols < p.tile_n) {  // the corpus's last tile: padding columns never qualify
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (b * 32 + j >= ncols) v[b][j] = -INFINITY;
        }
        float m = fmaxf(s1_tree_max32(v[0]), s1_tree_max32(v[1]));
        if (p.tile_n == 128) m = fmaxf(m, fmaxf(s1_tree_max32(v[2]), s1_tree_max32(v[3])));
        if (p.sample) {  // pre-pass: tile maxima only (distinct tokens of disjoint tiles)
          if (valid) p.tmax[(size_t)t * p.R + r] = m;
          continue;
        }
        if (valid && m >= thr) {
          // rare: visit only the qualifying columns of each block
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (b * 32 >= ncols) break;
            uint32_t mask = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) mask |= (b * 32 + j < ncols && v[b][j] >= thr) ? (1u << j) : 0u;
            if (!mask) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) scratch[j * 128 + rl] = v[b][j];
            while (mask) {
              const int j = __ffs(mask) - 1;
              mask &= mask - 1;
              const float x = scratch[j * 128 + rl];
              if (!(x >= thr)) continue;  // thr rose since the mask was built
              if (cnt < p.cap) mylist[cnt++] = make_uint2(__float_as_uint(x), (uint32_t)(tb + b * 32 + j));
              else ovf = true;
              if (ntop < p.kp || x > theta) {
                int s = ntop < p.kp ? ntop : p.kp - 1;
                while (s > 0 && tops[(s - 1) * 128 + rl] < x) {
                  tops[s * 128 + rl] = tops[(s - 1) * 128 + rl];
                  --s;
                }
                tops[s * 128 + rl] = x;
                if (ntop < p.kp) ++ntop;
                if (ntop == p.kp) {
                  theta = tops[(p.kp - 1) * 128 + rl];
                  thr = fmaxf(theta, gtheta) - eps2;
                }
              }
            }
          }
        }
      }
      if (valid && !p.sample) {
        p.cnt[(size_t)item * 128 + rl] = cnt;
        float* tv = p.topv + ((size_t)item * 128 + rl) * p.kp;
        for (int s = 0; s < p.kp; ++s) tv[s] = s < ntop ? tops[s * 128 + rl] : -INFINITY;
        if (ovf) atomicOr(p.status, 1);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<S1_ACC * S1_TILE>(tmem_base);
  }
}

constexpr int S1R_THREADS = 512;

// k-th largest (1-based) of n floats in shared memory: MSB-first radix select on order-preserving keys,
// 8 bits per pass (4 passes, 256-bin shared histogram). Every thread of the CTA returns the value.
__device__ float block_kth_largest(const float* sv, int n, int k, unsigned int* hist, unsigned int* bc) {
  unsigned int prefix = 0u, mask = 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned int key = ord_key(sv[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns bins [8l, 8l + 8); suffix sums from the top bin down
      unsigned int c[8], tot = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[lane * 8 + j];
        tot += c[j];
      }
      unsigned int incl = tot;  // inclusive suffix sum over lanes >= this one
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += y;
      }
      const unsigned int above = incl - tot;  // count in bins owned by higher lanes
      const unsigned int kk = (unsigned int)k;
      if (above < kk && kk <= above + tot) {  // the k-th largest falls in this lane's bins
        unsigned int acc = above;
        int d = 7;
        for (; d > 0; --d) {
          if (acc + c[d] >= kk) break;
          acc += c[d];
        }
        bc[0] = (unsigned int)(lane * 8 + d);
        bc[1] = kk - acc;
      }
    }
    __syncthreads();
    prefix |= bc[0] << shift;
    mask |= 255u << shift;
    k = (int)bc[1];
    __syncthreads();
  }
  return ord_val(prefix);
}

// gthr[r] = key of the k'-th largest pre-pass tile maximum of row r: k' distinct corpus tokens reach it,
// so it is a lower bound on the global k'-th value (0 = no bound when fewer than k' tiles were sampled)
__global__ void __launch_bounds__(S1R_THREADS) stage1_seed_kernel(S1Params p) {
  extern __shared__ __align__(16) uint8_t sd_smem[];
  __shared__ unsigned int hist[256], bc[2];
  float* sv = reinterpret_cast<float*>(sd_smem);
  const int64_t r = blockIdx.x;
  for (int i = threadIdx.x; i < p.NS; i += S1R_THREADS) sv[i] = p.tmax[(size_t)i * p.R + r];
  __syncthreads();
  const float x = p.kp <= p.NS ? block_kth_largest(sv, p.NS, p.kp, hist, bc) : -INFINITY;
  if (threadIdx.x == 0) p.gthr[r] = x > -INFINITY ? ord_key(x) : 0u;
}

template <typename T>
__global__ void __launch_bounds__(S1R_THREADS)
    stage1_refine_kernel(const T* __restrict__ q, const T* __restrict__ d, S1Params p, int dim, int clamp,
                         int64_t* __restrict__ nb_tok, double* __restrict__ nb_val) {
  extern __shared__ __align__(16) uint8_t rf_smem[];
  __shared__ int n_f;
  __shared__ int ovf;
  __shared__ unsigned int hist[256], bc[2];
  const int64_t r = blockIdx.x;
  const int rb = (int)(r / 128), rl = (int)(r % 128);
  const int n = p.P * p.kp;
  float* sv = reinterpret_cast<float*>(rf_smem);                  // [P * kp] (<= 148 * 256)
  uint64_t* fkey = reinterpret_cast<uint64_t*>(rf_smem);          // reused after the threshold: [S1_FCAP]
  uint32_t* ftok = reinterpret_cast<uint32_t*>(fkey + S1_FCAP);   // [S1_FCAP]
  float* qs = reinterpret_cast<float*>(ftok + S1_FCAP);           // [dim]
  if (threadIdx.x == 0) {
    n_f = 0;
    ovf = 0;
  }
  for (int i = threadIdx.x; i < n; i += S1R_THREADS) {
    const int it = rb * p.P + i / p.kp;
    sv[i] = p.topv[((size_t)it * 128 + rl) * p.kp + i % p.kp];
  }
  __syncthreads();
  const float thr = block_kth_largest(sv, n, p.kp, hist, bc) - 2.0f * p.eps[r];
  __syncthreads();  // sv is overwritten below
  // one item's list per warp lane-strided (lists are short after the pre-pass; items are many)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pp = warp; pp < p.P; pp += S1R_THREADS / 32) {
    const size_t it = (size_t)rb * p.P + pp;
    const int c = p.cnt[it * 128 + rl];
    const uint2* lst = p.ent + (it * 128 + rl) * p.cap;
    for (int e = lane; e < c; e += 32) {
      const uint2 u = lst[e];
      if (__uint_as_float(u.x) >= thr) {
        const int s = atomicAdd(&n_f, 1);
        if (s < S1_FCAP) ftok[s] = u.y;
        else ovf = 1;
      }
    }
  }
  for (int k = threadIdx.x; k < dim; k += S1R_THREADS) qs[k] = Elem<T>::to_f(q[r * dim + k]);
  __syncthreads();
  const int nf = n_f < S1_FCAP ? n_f : S1_FCAP;
  int SF = 32;
  while (SF < nf) SF <<= 1;
  for (int i = threadIdx.x; i < SF; i += S1R_THREADS) {
    if (i < nf) {
      const T* e = d + (size_t)ftok[i] * dim;
      double acc = 0.0;
      for (int k = 0; k < dim; ++k) acc = fma(Elem<T>::to_d(__ldg(e + k)), (double)qs[k], acc);
      if (clamp) acc = acc > 0.0 ? acc : 0.0;
      fkey[i] = desc_key_f64(acc);
    } else {
      fkey[i] = ~0ull;
      ftok[i] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  for (int k = 2; k <= SF; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < SF; i += S1R_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = fkey[i], b2 = fkey[ixj];
          const uint32_t ia = ftok[i], ib = ftok[ixj];
          const bool a_gt = a > b2 || (a == b2 && ia > ib);
          if (((i & k) == 0) == a_gt) {
            fkey[i] = b2;
            fkey[ixj] = a;
            ftok[i] = ib;
            ftok[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < p.kp; i += S1R_THREADS) {
    const uint64_t u = ~fkey[i];
    const uint64_t bits = (u & 0x8000000000000000ull) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
    const double v = __longlong_as_double((long long)bits);
    nb_tok[r * p.kp + i] = ftok[i];
    nb_val[r * p.kp + i] = v;
    if (i == p.kp - 1 && clamp && v == 0.0) atomicOr(p.status, 2);  // zero ties: corpus order decides
  }
  if (threadIdx.x == 0 && (ovf || nf < p.kp)) atomicOr(p.status, 1);
}

struct TcPlan {
  int RB, P, NT, kblocks, stages, items, cap, tile_n;
  int ns_stride, ns;  // threshold pre-pass: tile stride and sampled tiles (0 = no pre-pass)
  size_t smem, o_eps, o_gthr, o_cnt, o_ent, o_topv, o_tmax, total;
};

// shared memory of the scan for k': query block + sorted tops + scratch + >= 2 stages of tiles (plan_tc)
static bool tc_fits(int dim, int kp) {
  const size_t kblocks = (size_t)(dim + 63) / 64;
  const size_t fixed = 1024 + kblocks * 16384 + 4 * (size_t)kp * 128 + 4 * 32 * 128 + 8 * 32;
  if (fixed >= 227 * 1024) return false;
  const size_t budget = 227 * 1024 - fixed;
  const size_t tile_n = budget / (kblocks * 16384) >= 3 ? 128 : 64;
  return budget / (kblocks * tile_n * 128) >= 2;
}

static bool tc_eligible(const cbx_batch* b, int kp) {
  return (b->dtype == CBX_F16 || b->dtype == CBX_BF16) && b->dim % 8 == 0 && b->dim <= 256 && kp <= S1_MAX_KP &&
         tc_fits(b->dim, kp) && b->n_d_tokens >= S1_MIN_TOKENS && b->n_d_tokens < (int64_t(1) << 31) &&
         b->n_q_tokens < (int64_t(1) << 24);
}

static int plan_tc(const cbx_batch* b, int kp, TcPlan& t) {
  const int64_t R = b->n_q_tokens, Tn = b->n_d_tokens;
  t.RB = (int)((R + 127) / 128);
  t.kblocks = (b->dim + 63) / 64;
  const size_t qb = (size_t)t.kblocks * 16384;
  const size_t fixed = 1024 + qb + 4 * (size_t)kp * 128 + 4 * 32 * 128 + 8 * 32;
  const size_t budget = 227 * 1024 - fixed;
  t.tile_n = budget / ((size_t)t.kblocks * 16384) >= 3 ? 128 : 64;  // keep >= 3 stages in flight
  const size_t sb = (size_t)t.kblocks * t.tile_n * 128;
  t.stages = (int)std::min<size_t>(S1_MAX_STAGES, budget / sb);
  if (t.stages < 2) return fail(CBX_EINVAL, "stage-1 scan: tile does not fit shared memory");
  t.NT = (int)((Tn + t.tile_n - 1) / t.tile_n);
  const int G = sm_count();
  t.P = t.RB >= G ? 1 : std::min(t.NT, (G + t.RB - 1) / t.RB);
  t.items = t.RB * t.P;
  t.smem = fixed + (size_t)t.stages * sb;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  t.o_eps = take(4 * (size_t)R);
  t.o_gthr = take(4 * (size_t)R);
  t.o_cnt = take(4 * (size_t)t.items * 128);
  // expected appends per list ~ kp * (1 + ln(tokens per item / kp)); overflow falls back to SIMT
  t.cap = std::min(4096, std::max(256, 12 * kp));
  t.o_ent = take(8 * (size_t)t.items * 128 * t.cap);
  t.o_topv = take(4 * (size_t)t.items * 128 * kp);
  // pre-pass sample: ~16 tiles per SM, at most 4096 tiles and 16 MB of tile maxima
  int64_t want = std::min<int64_t>({(int64_t)G * 16, 4096, ((int64_t)1 << 22) / std::max<int64_t>(R, 1)});
  t.ns_stride = want > 0 ? (int)(t.NT / want) : 0;
  t.ns = t.ns_stride >= 2 ? (t.NT + t.ns_stride - 1) / t.ns_stride : 0;
  if (t.ns < 4 * kp) t.ns = 0;
  t.o_tmax = take(4 * (size_t)std::max(t.ns, 1) * R);
  t.total = o;
  return CBX_OK;
}

template <typename T>
static int run_tc(const cbx_batch* b, int kp, float norm_max, int64_t* nb_tok, double* nb_val, int* status,
                  uint8_t* ws, cudaStream_t st) {
  TcPlan t;
  int rc = plan_tc(b, kp, t);
  if (rc) return rc;
  S1Params p;
  p.R = b->n_q_tokens;
  p.T = b->n_d_tokens;
  p.RB = t.RB;
  p.P = t.P;
  p.NT = t.NT;
  p.kp = kp;
  p.cap = t.cap;
  p.kblocks = t.kblocks;
  p.stages = t.stages;
  p.tile_n = t.tile_n;
  p.idesc = ptx::idesc_f16(b->dtype == CBX_BF16, 128, (uint32_t)t.tile_n);
  p.q_slot_bytes = (uint32_t)(t.kblocks * 16384);
  p.stage_bytes = (uint32_t)(t.kblocks * t.tile_n * 128);
  p.eps = reinterpret_cast<float*>(ws + t.o_eps);
  p.gthr = reinterpret_cast<unsigned int*>(ws + t.o_gthr);
  p.cnt = reinterpret_cast<int32_t*>(ws + t.o_cnt);
  p.ent = reinterpret_cast<uint2*>(ws + t.o_ent);
  p.topv = reinterpret_cast<float*>(ws + t.o_topv);
  p.tmax = reinterpret_cast<float*>(ws + t.o_tmax);
  p.status = status;
  CUtensorMap tm_d, tm_q;
  rc = make_tmap(&tm_d, b->d_tokens, b->dtype, b->n_d_tokens, b->dim, (uint32_t)t.tile_n);
  if (rc) return rc;
  rc = make_tmap(&tm_q, b->q_tokens, b->dtype, b->n_q_tokens, b->dim, 128);
  if (rc) return rc;
  stage1_eps_kernel<<<(unsigned)((p.R + 7) / 8), 256, 0, st>>>(b->q_tokens, b->dtype, p.R, b->dim, norm_max,
                                                               const_cast<float*>(p.eps));
  CBX_LAUNCH_CHECK("stage1_eps_kernel launch");
  CBX_CUDA_CHECK(cudaFuncSetAttribute(stage1_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem));
  const int G = sm_count();
  // threshold pre-pass over every stride-th tile: seeds each row's filter with the k'-th largest sampled
  // tile maximum, so the main scan appends / inserts almost only true contenders
  if (t.ns) {
    S1Params ps = p;
    ps.sample = 1;
    ps.stride = t.ns_stride;
    ps.NS = t.ns;
    ps.P = t.RB >= G ? 1 : std::min(ps.NS, (G + t.RB - 1) / t.RB);
    stage1_scan_kernel<<<std::min(t.RB * ps.P, G), S1_THREADS, t.smem, st>>>(tm_d, tm_q, ps);
    CBX_LAUNCH_CHECK("stage1_scan_kernel (pre-pass) launch");
    CBX_CUDA_CHECK(cudaFuncSetAttribute(stage1_seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * ps.NS));
    stage1_seed_kernel<<<(unsigned)p.R, S1R_THREADS, 4 * ps.NS, st>>>(ps);
    CBX_LAUNCH_CHECK("stage1_seed_kernel launch");
  } else {
    CBX_CUDA_CHECK(cudaMemsetAsync(p.gthr, 0, 4 * (size_t)p.R, st));  // key 0: no seed
  }
  p.sample = 0;
  p.stride = 1;
  p.NS = t.NT;
  stage1_scan_kernel<<<std::min(t.items, G), S1_THREADS, t.smem, st>>>(tm_d, tm_q, p);
  CBX_LAUNCH_CHECK("stage1_scan_kernel launch");
  const size_t rsmem = std::max<size_t>(4 * (size_t)t.P * kp, 12 * (size_t)S1_FCAP + 4 * (size_t)b->dim);
  CBX_CUDA_CHECK(cudaFuncSetAttribute(stage1_refine_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
  stage1_refine_kernel<T><<<(unsigned)p.R, S1R_THREADS, rsmem, st>>>(
      static_cast<const T*>(b->q_tokens), static_cast<const T*>(b->d_tokens), p, b->dim, b->clamp_negative, nb_tok,
      nb_val);
  CBX_LAUNCH_CHECK("stage1_refine_kernel launch");
  return CBX_OK;
}

// ============================================================ corpus norm
template <typename T>
__global__ void token_norm_max_kernel(const T* __restrict__ x, int64_t n, int dim, unsigned int* out_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  float best = 0.0f;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5); r < n; r += warps) {
    double s = 0.0;
    for (int k = lane; k < dim; k += 32) {
      const double v = Elem<T>::to_d(x[r * dim + k]);
      s += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    best = fmaxf(best, __double2float_ru(sqrt(s)));
  }
  if (lane == 0) atomicMax(out_bits, __float_as_uint(best));  // non-negative floats order like their bits
}

static int resolve_path(const cbx_batch* b, int kp, int path) {
  if (path == CBX_PATH_AUTO) return tc_eligible(b, kp) ? CBX_PATH_TC : CBX_PATH_SIMT;
  return path;
}

static int check_stage1(const cbx_batch* b, int kp) {
  if (!b) return fail(CBX_EINVAL, "batch descriptor is NULL");
  if (kp < 1) return fail(CBX_EINVAL, "k_prime must be at least 1, got " + std::to_string(kp));
  if (b->n_q_tokens < 1 || b->n_d_tokens < 1) return fail(CBX_EINVAL, "stage-1 scan needs query rows and corpus tokens");
  if (kp > b->n_d_tokens) return fail(CBX_EINVAL, "k_prime exceeds the corpus token count");
  if (kp > 8192) return fail(CBX_EINVAL, "k_prime > 8192 is not supported");
  if (b->n_q_tokens > 65535) return fail(CBX_EINVAL, "stage-1 scan: at most 65535 query rows per call");
  if (b->dim <= 0 || dtype_size(b->dtype) == 0) return fail(CBX_EINVAL, "bad dim / dtype");
  if (!b->q_tokens || !b->d_tokens) return fail(CBX_EINVAL, "token buffers are NULL");
  return CBX_OK;
}

}  // namespace cbx

using namespace cbx;

extern "C" {

size_t cbx_stage1_workspace_bytes(const cbx_batch* b, int k_prime, int path) {
  if (check_stage1(b, k_prime)) return 0;
  path = resolve_path(b, k_prime, path);
  if (path == CBX_PATH_TC) {
    TcPlan t;
    if (plan_tc(b, k_prime, t)) return 0;
    return t.total;
  }
  return plan_simt(b->n_q_tokens, b->n_d_tokens, k_prime).total;
}

int cbx_stage1_topk(const cbx_batch* b, int k_prime, int path, float corpus_norm_max, int64_t* nb_tok,
                    double* nb_val, int* status, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_stage1(b, k_prime);
  if (rc) return rc;
  if (!nb_tok || !nb_val || !status) return fail(CBX_EINVAL, "stage-1 output buffers are NULL");
  path = resolve_path(b, k_prime, path);
  if (path != CBX_PATH_TC && path != CBX_PATH_SIMT) return fail(CBX_EINVAL, "unknown stage-1 path");
  if (path == CBX_PATH_TC && !tc_eligible(b, k_prime))
    return fail(CBX_EINVAL, "stage-1 tcgen05 path needs f16/bf16, dim % 8 == 0, dim <= 256, k_prime <= 64 and a "
                            "corpus of at least 8192 tokens");
  if (path == CBX_PATH_TC && !(corpus_norm_max > 0.0f && corpus_norm_max < INFINITY))
    return fail(CBX_EINVAL, "stage-1 tcgen05 path needs the corpus max token norm (cbx_token_norm_max)");
  if (ws_bytes < cbx_stage1_workspace_bytes(b, k_prime, path)) return fail(CBX_EINVAL, "stage-1 workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  CBX_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
  if (path == CBX_PATH_TC) {
    if (b->dtype == CBX_F16) return run_tc<__half>(b, k_prime, corpus_norm_max, nb_tok, nb_val, status, w, st);
    return run_tc<__nv_bfloat16>(b, k_prime, corpus_norm_max, nb_tok, nb_val, status, w, st);
  }
  switch (b->dtype) {
    case CBX_F32: return run_simt<float>(b, k_prime, nb_tok, nb_val, w, st);
    case CBX_F64: return run_simt<double>(b, k_prime, nb_tok, nb_val, w, st);
    case CBX_F16: return run_simt<__half>(b, k_prime, nb_tok, nb_val, w, st);
    case CBX_BF16: return run_simt<__nv_bfloat16>(b, k_prime, nb_tok, nb_val, w, st);
  }
  return fail(CBX_EINVAL, "unknown dtype");
}

int cbx_token_norm_max(const void* tokens, int64_t n_tokens, int dim, int dtype, float* out, void* stream) {
  if (!tokens || !out || n_tokens < 1 || dim < 1) return fail(CBX_EINVAL, "token_norm_max: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CBX_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(float), st));
  unsigned int* bits = reinterpret_cast<unsigned int*>(out);
  const int grid = (int)std::min<int64_t>((n_tokens + 7) / 8, (int64_t)sm_count() * 8);
  switch (dtype) {
    case CBX_F32: token_norm_max_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(tokens), n_tokens, dim, bits); break;
    case CBX_F64: token_norm_max_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(tokens), n_tokens, dim, bits); break;
    case CBX_F16: token_norm_max_kernel<__half><<<grid, 256, 0, st>>>(static_cast<const __half*>(tokens), n_tokens, dim, bits); break;
    case CBX_BF16:
      token_norm_max_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(tokens), n_tokens, dim, bits);
      break;
    default: return fail(CBX_EINVAL, "unknown dtype");
  }
  CBX_LAUNCH_CHECK("token_norm_max_kernel launch");
  return CBX_OK;
}

}  // extern "C"
