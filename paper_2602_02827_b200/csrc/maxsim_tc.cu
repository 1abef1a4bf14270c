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

#ifndef CBX_TC_EPI_WARP0
#define CBX_TC_EPI_WARP0 4  // first of the four epilogue warps (warp % 4 = its TMEM lane quarter)
#endif
constexpr int TC_THREADS = (CBX_TC_EPI_WARP0 + 4) * 32;
constexpr int TC_EPI_WARP0 = CBX_TC_EPI_WARP0;
static_assert(TC_EPI_WARP0 % 4 == 0, "epilogue warps must cover TMEM lane quarters 0..3 in order");
constexpr int TC_ACC_BUFS = 4;      // accumulator barrier pairs (a ring of four, whatever the number of accumulators)
constexpr int TC_TMEM_COLS = 512;   // all of TMEM: 4 accumulators of 128 columns, or 2 of 256
constexpr int TC_MAX_TILE_N = 256;
#ifndef CBX_TC_TILE256
#define CBX_TC_TILE256 1  // contiguous batches with d <= 128: 256-token tiles (half the per-tile work per byte)
#endif
#ifndef CBX_PK_TILE_N
#define CBX_PK_TILE_N 128  // packed-mode tile height (build knob; 64 measured much slower)
#endif
static_assert(CBX_PK_TILE_N == 32 || CBX_PK_TILE_N == 64 || CBX_PK_TILE_N == 128,
              "packed tile height must be 32, 64 or 128 rows (8-row TMA boxes d[k8], whole pack slots)");
constexpr int TC_MAX_STAGES = 8;
#ifndef CBX_PACK_ALIGN
#define CBX_PACK_ALIGN 32
#endif
#ifndef CBX_PK_PRODUCERS
#define CBX_PK_PRODUCERS 3  // packed-mode TMA issuer warps: warp 0 plus warps 2.. (A/B knob for tools/mkvar.sh)
#endif
static_assert(CBX_PK_PRODUCERS >= 1 && CBX_PK_PRODUCERS <= CBX_TC_EPI_WARP0 - 1, "producers must end before the epilogue");
constexpr int TC_PACK = CBX_PACK_ALIGN;  // packed-mode row granularity (power of two, >= 8)
static_assert(TC_PACK >= 8 && (TC_PACK & (TC_PACK - 1)) == 0 && CBX_PK_TILE_N % TC_PACK == 0,
              "packed tiles must hold whole pack slots");

struct TcParams {
  const int64_t* q_tok_off;
  const int64_t* d_tok_off;   // token offsets; in packed mode the 8-aligned packed starts
  const int64_t* q_doc_off;
  float* scores;
  // packed mode: document j is rows [src_row[j], src_row[j] + doc_len[j]) of a corpus tensor and is
  // laid out in the tile stream at packed rows [d_tok_off[j], d_tok_off[j] + doc_len[j]), 8-row aligned
  int32_t packed;
  const int64_t* src_row;
  const int32_t* doc_len;
  const int64_t* n_tokens_dev;  // packed mode: total packed rows (d_tok_off[n_docs]) read on the device
  // packed mode with dim % 64 == 0: stages interleave the K blocks per 8-row group so one 4-D TMA box
  // carries all K blocks of a row range (TmapSet::pk); corpus_rows bounds those maps, k8 = 8-row 2-D map
  int32_t ilv;
  int32_t k8;
  int64_t corpus_rows;
  int64_t n_queries;
  int64_t n_docs;
  int64_t n_tokens;      // total document tokens (partitioned evenly over the CTAs)
  uint32_t idesc;
  int32_t tile_n;
  int32_t kblocks;       // ceil(dim / 64)
  int32_t lqp;           // query rows per replica (max Lq rounded up to 32)
  int32_t nq;            // TMEM lane quadrants per replica (lqp / 32)
  int32_t rep;           // query replicas in the 128-row A operand (4 / nq, 1 if nq == 3)
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

// Static balanced partition: CTA b owns the documents whose first token lies in
// [b * n_tokens / G, (b + 1) * n_tokens / G); its "chunks" are that document
// range cut at query boundaries, visited in order. Every role walks the same
// sequence, so no scheduling state is exchanged.
struct ChunkCursor {
  int64_t doc, doc_hi, q;
  __device__ __forceinline__ void init(TcParams& p) {
    if (p.packed) p.n_tokens = *p.n_tokens_dev;
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t x0 = (int64_t)((__int128)p.n_tokens * b / G);
    const int64_t x1 = (int64_t)((__int128)p.n_tokens * (b + 1) / G);
    doc = lower_bound_start(p.d_tok_off, 0, p.n_docs, x0);
    doc_hi = lower_bound_start(p.d_tok_off, doc, p.n_docs, x1);
    // query owning `doc`: last q with q_doc_off[q] <= doc
    int64_t lo = 0, hi = p.n_queries;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(p.q_doc_off + mid) <= doc) lo = mid;
      else hi = mid;
    }
    q = lo;
  }
  __device__ __forceinline__ bool next(const TcParams& p, ChunkInfo& c) {
    if (doc >= doc_hi) return false;
    int64_t qe;
    while ((qe = __ldg(p.q_doc_off + q + 1)) <= doc) ++q;
    c.doc0 = doc;
    c.doc1 = qe < doc_hi ? qe : doc_hi;
    doc = c.doc1;
    c.cs = __ldg(p.d_tok_off + c.doc0);
    c.ce = __ldg(p.d_tok_off + c.doc1);
    c.q_tok0 = __ldg(p.q_tok_off + q);
    c.lq = (int32_t)(__ldg(p.q_tok_off + q + 1) - c.q_tok0);
    c.ntiles = (int32_t)((c.ce - c.cs + p.tile_n - 1) / p.tile_n);
    return true;
  }
};

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// max of 32 register values (FMNMX3 tree)
__device__ __forceinline__ float max32(const float (&v)[32]) {
  float a[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) a[i] = fmax3f(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  a[10] = fmaxf(v[30], v[31]);
  float b0 = fmax3f(a[0], a[1], a[2]), b1 = fmax3f(a[3], a[4], a[5]), b2 = fmax3f(a[6], a[7], a[8]);
  float b3 = fmaxf(a[9], a[10]);
  return fmaxf(fmax3f(b0, b1, b2), b3);
}

// max of v[j] for s <= j < e (s, e warp-uniform), starting from m
__device__ __forceinline__ float masked_max(const float (&v)[32], int s, int e, float m) {
  const uint32_t bits = (e >= 32 ? 0xFFFFFFFFu : ((1u << e) - 1u)) & ~((1u << s) - 1u);
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (bits & (1u << j)) m = fmaxf(m, v[j]);
  return m;
}

// tensor maps: doc tiles of box heights tile_n >> k (k = 0..4; packed mode uses all of them to lay
// documents out at 8-row granularity) and the query rows
// pk[k][r]: packed interleaved mode, 4-D view {64 cols, 8 rows, kblocks, 8-row groups} of the corpus
// from row r on, boxes of (tile_n >> k) rows x every K block
static_assert(TC_PACK >= 32, "interleaved packed maps cover box heights tile_n >> {0,1,2} only");
struct TmapSet {
  CUtensorMap d[5];
  CUtensorMap q;
  CUtensorMap pk[3][8];
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    maxsim_tc_kernel(const __grid_constant__ TmapSet tm, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_slot = smem;                                    // kblocks x (128 rows x 128 B)
  uint8_t* stages = smem + p.q_slot_bytes;                   // stages x stage_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)p.stages * p.stage_bytes);
  uint64_t* full = bars;                                     // [TC_MAX_STAGES]
  uint64_t* empty = bars + TC_MAX_STAGES;                    // [TC_MAX_STAGES]
  uint64_t* qfull = bars + 2 * TC_MAX_STAGES;                // [1]
  uint64_t* qempty = qfull + 1;                              // [1]
  uint64_t* tfull = qempty + 1;                              // [4]
  uint64_t* tempty = tfull + TC_ACC_BUFS;                    // [4]
  uint64_t* cfull = tempty + TC_ACC_BUFS;                    // [4] carry published
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(cfull + TC_ACC_BUFS);
  float* carry = reinterpret_cast<float*>(bars + 64);        // [4 slots][4 warps][32]
  float* part = carry + 4 * 4 * 32;                          // [2 parity][4 quads][TC_MAX_TILE_N]
  int64_t* part_doc = reinterpret_cast<int64_t*>(part + 2 * 4 * TC_MAX_TILE_N);  // [2][2 groups][TC_MAX_TILE_N]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(qfull, 1);
    ptx::mbar_init(qempty, 1);
    for (int s = 0; s < TC_ACC_BUFS; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], p.nq);
      ptx::mbar_init(&cfull[s], p.nq);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    for (int k = 0; k < 5; ++k) ptx::prefetch_tmap(&tm.d[k]);
    ptx::prefetch_tmap(&tm.q);
  }
  if (warp == 1) ptx::tmem_alloc<TC_TMEM_COLS>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0 || (p.packed && warp >= 2 && warp <= CBX_PK_PRODUCERS && warp - 1 < p.stages)) {
    // ------------------------------------------------------------ TMA producers (lane 0 issues)
    // Warp 0 loads the query and, in packed mode, shares the document tiles round-robin with warps 2
    // and 3 (packed tiles need several small boxes each; three issuers keep the ring full).
    // a producer may only run one ring lap ahead of the slowest one: np <= stages keeps every
    // empty-barrier parity wait unambiguous
    const int np = p.packed ? (p.stages < CBX_PK_PRODUCERS ? p.stages : CBX_PK_PRODUCERS) : 1;
    const int pi = warp == 0 ? 0 : warp - 1;
    uint32_t qphase = 0, tg = 0;
    const uint64_t pol = ptx::policy_evict_first();
    ChunkCursor cur;
    cur.init(p);
    ChunkInfo c;
    while (cur.next(p, c)) {
      if (pi == 0 && lane == 0) {
        // one query slot: reload only after every MMA of the previous chunk retired
        ptx::mbar_wait(qempty, qphase ^ 1);
        ptx::mbar_arrive_expect_tx(qfull, (uint32_t)(p.rep * p.kblocks * p.lqp * 128));
        for (int g = 0; g < p.rep; ++g)
          for (int kb = 0; kb < p.kblocks; ++kb)
            ptx::tma_load_2d(q_slot + kb * 16384 + g * p.lqp * 128, &tm.q, qfull, kb * 64, (int32_t)c.q_tok0);
      }
      qphase ^= 1;
      // packed mode: metadata of 32 documents per lane window (packed start, corpus row, length)
      int64_t jd = c.doc0, win = c.doc0;
      int64_t w_pk = 0, w_src = 0;
      int32_t w_len = 0;
      if (p.packed && win + lane < c.doc1) {
        w_pk = __ldg(p.d_tok_off + win + lane);
        w_src = __ldg(p.src_row + win + lane);
        w_len = __ldg(p.doc_len + win + lane);
      }
      for (int t = 0; t < c.ntiles; ++t, ++tg) {
        const int64_t r0 = c.cs + (int64_t)t * p.tile_n;
        const int64_t r1 = c.ce - r0 < p.tile_n ? c.ce : r0 + p.tile_n;
        const bool mine = (int)(tg % (uint32_t)np) == pi;
        const uint32_t stage = tg % (uint32_t)p.stages, phase = (tg / (uint32_t)p.stages) & 1u;
        if (lane == 0 && mine) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], p.packed ? (uint32_t)((r1 - r0) * 128 * p.kblocks) : p.stage_bytes);
        }
        __syncwarp();
        uint8_t* dst = stages + (size_t)stage * p.stage_bytes;
        if (!p.packed) {
          if (lane == 0 && mine)
            for (int kb = 0; kb < p.kblocks; ++kb)
              ptx::tma_load_2d_hint(dst + kb * p.tile_n * 128, &tm.d[0], &full[stage], kb * 64, (int32_t)r0, pol);
        } else {
          // every document overlapping packed rows [r0, r1): boxes of 8 * 2^k rows at 8-aligned smem rows
          while (true) {
            if (jd - win >= 32) {
              win += 32;
              w_pk = w_src = 0;
              w_len = 0;
              if (win + lane < c.doc1) {
                w_pk = __ldg(p.d_tok_off + win + lane);
                w_src = __ldg(p.src_row + win + lane);
                w_len = __ldg(p.doc_len + win + lane);
              }
            }
            if (jd >= c.doc1) break;
            const int sl = (int)(jd - win);
            const int64_t pk = __shfl_sync(0xffffffffu, w_pk, sl);
            if (pk >= r1) break;
            const int64_t src = __shfl_sync(0xffffffffu, w_src, sl);
            const int32_t len = __shfl_sync(0xffffffffu, w_len, sl);
            const int64_t pk_next = pk + ((len + TC_PACK - 1) & ~(TC_PACK - 1));
            const int64_t ov0 = pk > r0 ? pk : r0;
            const int64_t ov1 = pk_next < r1 ? pk_next : r1;
            if (lane == 0 && mine) {
              int64_t row = ov0, srow = src + (ov0 - pk);
              for (int k = 0; k < 5; ++k) {
                const int h = p.tile_n >> k;
                if (h < TC_PACK) break;
                while (ov1 - row >= h) {
                  if (p.ilv) {
                    // interleaved stage: 8-row groups of kblocks x 1 KB; one 4-D box (rows x all K blocks)
                    // through the map whose base is corpus row (srow & 7), unless the box reaches past that
                    // map's last whole 8-row group (corpus tail: 8-row 2-D boxes, zero-filled past the end)
                    uint8_t* bdst = dst + (row - r0) * 128 * p.kblocks;
                    const int ph = (int)(srow & 7);
                    const int64_t g = srow >> 3;
                    if (g + (h >> 3) <= ((p.corpus_rows - ph) >> 3)) {
                      ptx::tma_load_4d_hint(bdst, &tm.pk[k][ph], &full[stage], 0, 0, 0, (int32_t)g, pol);
                    } else {
                      for (int gi = 0; gi < (h >> 3); ++gi)
                        for (int kb = 0; kb < p.kblocks; ++kb)
                          ptx::tma_load_2d_hint(bdst + (gi * p.kblocks + kb) * 1024, &tm.d[p.k8], &full[stage],
                                                kb * 64, (int32_t)(srow + gi * 8), pol);
                    }
                  } else {
                    for (int kb = 0; kb < p.kblocks; ++kb)
                      ptx::tma_load_2d_hint(dst + kb * p.tile_n * 128 + (row - r0) * 128, &tm.d[k], &full[stage],
                                            kb * 64, (int32_t)srow, pol);
                  }
                  row += h;
                  srow += h;
                }
              }
            }
            if (pk_next > r1) break;  // document continues into the next tile
            ++jd;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, qphase = 0, tg = 0;
      ChunkCursor cur;
      cur.init(p);
      ChunkInfo c;
      const uint32_t q_addr = ptx::smem_u32(q_slot);
      const uint64_t ad0 = ptx::smem_desc_sw128(q_addr);
      while (cur.next(p, c)) {
        ptx::mbar_wait(qfull, qphase);
        qphase ^= 1;
        ptx::tc_fence_after();
        for (int t = 0; t < c.ntiles; ++t, ++tg) {
          // accumulators: 4 x 128 columns, or 2 x 256 for 256-token tiles; their barriers are a ring of four
          // indexed by the tile either way (a group of the epilogue meets every rep-th tile: a barrier shared
          // with another group's tiles would put its waiter two phases behind — parity aliasing)
          const uint32_t nacc = p.tile_n > 128 ? 2u : 4u;
          const uint32_t acc = tg & (nacc - 1);
          if (tg >= nacc) ptx::mbar_wait(&tempty[(tg - nacc) & 3], ((tg - nacc) >> 2) & 1);
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t b_addr = ptx::smem_u32(stages + (size_t)stage * p.stage_bytes);
          const uint32_t d_tmem = tmem_base + acc * (p.tile_n > 128 ? 256u : 128u);
          // descriptors advance by (byte offset >> 4) in their 14-bit start-address field
          // interleaved (packed) stages: K block kb is 1 KB into each 8-row group, groups kblocks KB apart
          const uint64_t bd0 = ptx::smem_desc_sw128(b_addr, p.ilv ? (uint32_t)p.kblocks * 1024u : 1024u);
          const uint32_t bstep = (uint32_t)(p.ilv ? 1024 : p.tile_n * 128) >> 4;
#pragma unroll
          for (int kb = 0; kb < 8; ++kb) {
            if (kb >= p.kblocks) break;
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              ptx::tc_mma_f16(d_tmem, ad0 + (uint64_t)(kb * 1024 + k4 * 2), bd0 + (uint64_t)(kb * bstep + k4 * 2),
                              p.idesc, (kb | k4) != 0);
          }
          ptx::tc_commit(&empty[stage]);
          ptx::tc_commit(&tfull[tg & 3]);
          if (++stage == (uint32_t)p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit(qempty);
      }
    }
  } else if (warp >= TC_EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    // The query sits in the A operand `rep` times (rows g*lqp ...), so every
    // TMEM lane group holds the same scores; group g (nq warps = nq lane
    // quadrants) takes the CTA's tiles with index % rep == g. A document
    // spanning tiles is stitched through a carry chain: each tile publishes
    // the running max of the document open at its end (slot tg % 4), the
    // next tile merges it into its head segment.
    const int quad = warp - TC_EPI_WARP0;
    const int nq = p.nq, rep = p.rep;
    const int grp = quad / nq, wig = quad - grp * nq;
    if (grp < rep) {
      const float init = p.clamp_negative ? 0.0f : -INFINITY;
      const uint32_t tmem_lane = (uint32_t)(quad * 32) << 16;
      uint32_t tg = 0, pb = 0;
      ChunkCursor cursor;
      cursor.init(p);
      ChunkInfo c;
      while (cursor.next(p, c)) {
        const bool lane_valid = wig * 32 + lane < c.lq;
        // window of document end offsets: ends[lane] = end of doc (win + lane); in packed mode the end
        // of the valid rows, the next document starting at the following multiple of 8
        const int64_t align = p.packed ? TC_PACK - 1 : 0;
        auto end_of = [&](int64_t d) -> int64_t {
          if (d >= c.doc1) return INT64_MAX;
          return p.packed ? __ldg(p.d_tok_off + d) + __ldg(p.doc_len + d) : __ldg(p.d_tok_off + d + 1);
        };
        int64_t win = c.doc0;
        int64_t ends = end_of(win + lane);
        int64_t ends_nx = end_of(win + 32 + lane);
        int64_t doc = c.doc0;
        int64_t prev_end = c.cs;
        for (int t = 0; t < c.ntiles; ++t, ++tg) {
          if ((int)(tg % (uint32_t)rep) != grp) continue;
          const uint32_t acc = tg & (p.tile_n > 128 ? 1u : 3u);
          ptx::mbar_wait(&tfull[tg & 3], (tg >> 2) & 1);
          ptx::tc_fence_after();
          const int64_t tb = c.cs + (int64_t)t * p.tile_n;
          const int ncols = (int)(c.ce - tb < p.tile_n ? c.ce - tb : p.tile_n);
          // the accumulator is read 128 columns at a time (the registers' worth); `vload(hf)` brings half hf
          float v[4][32];
          const uint32_t taddr = tmem_base + tmem_lane + acc * (p.tile_n > 128 ? 256u : 128u);
          auto vload = [&](int hf) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (hf * 128 + b * 32 < ncols) ptx::tmem_ld_32x32b_x32(taddr + hf * 128 + b * 32, v[b]);
            ptx::tmem_ld_wait();
            if ((hf + 1) * 128 >= ncols) {  // the last columns are out: hand the accumulator back
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) ptx::mbar_arrive(&tempty[tg & 3]);
            }
          };
          vload(0);

          // skip documents that ended before this tile (other groups' tiles)
          int64_t cur_end;
          while (true) {
            if (doc - win >= 32) {
              win += 32;
              ends = ends_nx;
              ends_nx = end_of(win + 32 + lane);
              continue;
            }
            cur_end = __shfl_sync(0xffffffffu, ends, (int)(doc - win));
            if (cur_end > tb) break;
            prev_end = cur_end;
            ++doc;
          }
          int64_t doc_start = (prev_end + align) & ~align;
          const bool head_before = doc_start < tb;
          const int64_t head_doc = doc;
          int nfin = 0;
          float* mypart = part + (pb * 4 + quad) * TC_MAX_TILE_N;
          int64_t* mydocs = part_doc + (pb * 2 + grp) * TC_MAX_TILE_N;
          auto finalize = [&](int64_t d, float val) {
            const float x = warp_sum(lane_valid ? val : 0.0f);
            if (nq == 1) {
              if (lane == 0) p.scores[d] = x;
            } else {
              if (lane == 0) {
                mypart[nfin] = x;
                if (wig == 0) mydocs[nfin] = d;
              }
            }
            ++nfin;
          };
          float cur = init, H = init;
          bool head_open = true;
          auto close_seg = [&]() {
            if (head_open) {
              H = cur;
              head_open = false;
            } else {
              finalize(doc, cur);
            }
            cur = init;
            prev_end = cur_end;
            doc_start = (prev_end + align) & ~align;
            ++doc;
            if (doc - win >= 32) {
              win += 32;
              ends = ends_nx;
              ends_nx = end_of(win + 32 + lane);
            }
            cur_end = __shfl_sync(0xffffffffu, ends, (int)(doc - win));
          };
          for (int hf = 0; hf * 128 < ncols; ++hf) {
          if (hf > 0) vload(hf);
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (hf * 128 + b * 32 >= ncols) break;
            const int64_t g0 = tb + hf * 128 + b * 32;  // stream row of this block's column 0
            const int nc = ncols - hf * 128 - b * 32 < 32 ? ncols - hf * 128 - b * 32 : 32;
            while (true) {
              const int64_t ds = doc_start - g0;
              if (ds >= nc) break;  // the current document starts after this block (packed padding)
              const int64_t de = cur_end - g0;
              const int s = ds > 0 ? (int)ds : 0;
              const int e = de < nc ? (int)de : nc;
              if (s == 0 && e == 32) cur = fmaxf(cur, max32(v[b]));
              else cur = masked_max(v[b], s, e, cur);
              if (de > nc) break;  // document continues past this block
              close_seg();
            }
          }
          }
          // carry chain: merge the previous tile's open document into this head
          float p_prev = init;
          if (tg > 0) {
            const uint32_t ps = (tg - 1) & 3;
            ptx::mbar_wait(&cfull[ps], ((tg - 1) >> 2) & 1);
            p_prev = carry[(ps * 4 + wig) * 32 + lane];
          }
          float p_new, head_final = 0.0f;
          if (head_open) {
            p_new = head_before ? fmaxf(p_prev, cur) : cur;
          } else {
            head_final = head_before ? fmaxf(p_prev, H) : H;
            p_new = cur;
          }
          carry[((tg & 3) * 4 + wig) * 32 + lane] = p_new;
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&cfull[tg & 3]);
          if (!head_open) finalize(head_doc, head_final);
          if (nq > 1) {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(nq * 32) : "memory");
            if (wig == 0) {
              for (int j = lane; j < nfin; j += 32) {
                float sacc = part[(pb * 4 + grp * nq) * TC_MAX_TILE_N + j];
                for (int w = 1; w < nq; ++w) sacc += part[(pb * 4 + grp * nq + w) * TC_MAX_TILE_N + j];
                p.scores[mydocs[j]] = sacc;
              }
            }
            pb ^= 1;
          }
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TC_TMEM_COLS>(tmem_base);
  }
}

// ----------------------------------------------------------------- document-tile scorer (resident corpus)
// The reranking service's scorer: the candidates of every query are scored in place in an HBM-resident
// corpus (colbandit/oracle.py:205-227 for candidate lists). A tile is up to TR consecutive rows of ONE
// document (TR = 256 for d <= 128, 128 for d <= 256), loaded where it lies by one TMA box per K block (box
// heights 8, 16, ..., TR rows: at most 7 rows of over-read per tile) and multiplied with N = ceil16(rows):
// no packed layout, no per-tile document walk in the producer, no segment logic in the epilogue. Same roles
// and barriers as maxsim_tc_kernel; a document longer than one tile hands its running max to the next tile
// through the carry chain. The producer and the MMA issuer are single instruction streams, and at ~100
// instructions per tile they — not HBM — bound the first version of this kernel (128-row tiles, ncu:
// profiles/r2_ncu_docs_v2_cfg2_lines.txt); 256-row tiles cut the tiles per document from 1.87 to 1.17 on cfg2.
constexpr int DT_MAX_ROWS = 256;
constexpr int DT_SLOTS = 16;  // tiles in flight (barrier pairs); their bytes share one ring
struct DocTmaps {
  CUtensorMap d[DT_MAX_ROWS / 8];  // d[h - 1]: boxes of 8 h rows x 64 columns
  CUtensorMap q;
};

// 32 documents of metadata per lane window, the next window loaded one window ahead
struct DocWindow {
  int64_t win, hi;
  int64_t src, src_nx;
  int32_t len, len_nx;
  const int64_t* src_row;
  const int32_t* doc_len;
  bool want_src;
  __device__ __forceinline__ void fetch(int64_t w, int lane, int64_t& s, int32_t& l) const {
    s = 0;
    l = 0;
    if (w + lane < hi) {
      l = __ldg(doc_len + w + lane);
      if (want_src) s = __ldg(src_row + w + lane);
    }
  }
  __device__ __forceinline__ void open(const TcParams& p, int64_t lo, int64_t hi_, int lane, bool with_src) {
    src_row = p.src_row;
    doc_len = p.doc_len;
    want_src = with_src;
    win = lo;
    hi = hi_;
    fetch(win, lane, src, len);
    fetch(win + 32, lane, src_nx, len_nx);
  }
  // warp-collective: move the window so that it holds document d (documents are visited in order)
  __device__ __forceinline__ void seek(int64_t d, int lane) {
    while (d - win >= 32) {
      win += 32;
      src = src_nx;
      len = len_nx;
      fetch(win + 32, lane, src_nx, len_nx);
    }
  }
  __device__ __forceinline__ int32_t length(int64_t d) const { return __shfl_sync(0xffffffffu, len, (int)(d - win)); }
  __device__ __forceinline__ int64_t source(int64_t d) const { return __shfl_sync(0xffffffffu, src, (int)(d - win)); }
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    maxsim_docs_kernel(const __grid_constant__ DocTmaps tm, TcParams p) {
  // Shared memory: the query operand, then ONE byte ring for the document tiles: a tile of h rows takes
  // ceil8(h) x 128 B per K block, placed right behind its predecessor (wrapping to 0 when it would cross the
  // end). Placement is a pure function of the tile sizes, so the MMA warp recomputes it; the producer alone
  // tracks what has been consumed (virtual ring positions of the tiles in flight, one per lane).
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_slot = smem;                                    // kblocks x (128 rows x 128 B)
  uint8_t* ring = smem + p.q_slot_bytes;                     // ring_bytes (+ 1 KB the last tile's MMA may over-read)
  const uint32_t C = (uint32_t)p.stages * p.stage_bytes;     // ring capacity (multiple of 1024)
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + C + 1024);
  uint64_t* full = bars;                                     // [DT_SLOTS]
  uint64_t* empty = bars + DT_SLOTS;                         // [DT_SLOTS]
  uint64_t* qfull = bars + 2 * DT_SLOTS;                     // [1]
  uint64_t* qempty = qfull + 1;                              // [1]
  uint64_t* tfull = qempty + 1;                              // [4]
  uint64_t* tempty = tfull + TC_ACC_BUFS;                    // [4]
  uint64_t* cfull = tempty + TC_ACC_BUFS;                    // [4] carry published
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(cfull + TC_ACC_BUFS);
  float* carry = reinterpret_cast<float*>(bars + 64);        // [4 slots][4 warps][32]
  float* part = carry + 4 * 4 * 32;                          // [2 parity][4 quads]
  static_assert(2 * DT_SLOTS + 2 + 3 * TC_ACC_BUFS + 1 <= 64, "barrier block");
  static_assert(DT_SLOTS <= 32, "one lane per tile in flight");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int TR = p.tile_n;                     // tile rows: 128 or 256
  // TMEM accumulators: 4 x 128 or 2 x 256 columns. The accumulator barriers are always a ring of four
  // (index tg & 3): with rep = 4 a group meets every fourth tile, and a barrier that also completed for
  // another group's tile in between would put the waiter two phases behind (parity aliasing).
  const uint32_t nacc = 512u / (uint32_t)TR, accmask = nacc - 1u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < DT_SLOTS; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(qfull, 1);
    ptx::mbar_init(qempty, 1);
    for (int s = 0; s < TC_ACC_BUFS; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], p.nq);
      ptx::mbar_init(&cfull[s], p.nq);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 0 && lane < TR / 8) ptx::prefetch_tmap(&tm.d[lane]);
  if (warp == 2 && lane == 0) ptx::prefetch_tmap(&tm.q);
  if (warp == 1) ptx::tmem_alloc<512>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // every lane runs the same stream (no divergent sections); lane 0 arms the barriers and issues the copies
    uint32_t qphase = 0, tg = 0, tail = 0, off = 0;
    uint64_t vpos = 0, vs = 0;  // vs: virtual ring position of the tile in flight in slot `lane`
    const uint64_t pol = ptx::policy_evict_first();
    ChunkCursor cur;
    cur.init(p);
    ChunkInfo c;
    while (cur.next(p, c)) {
      ptx::mbar_wait(qempty, qphase ^ 1);
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(qfull, (uint32_t)(p.rep * p.kblocks * p.lqp * 128));
        for (int g = 0; g < p.rep; ++g)
          for (int kb = 0; kb < p.kblocks; ++kb)
            ptx::tma_load_2d(q_slot + kb * 16384 + g * p.lqp * 128, &tm.q, qfull, kb * 64, (int32_t)c.q_tok0);
      }
      qphase ^= 1;
      DocWindow w;
      w.open(p, c.doc0, c.doc1, lane, true);
      for (int64_t d = c.doc0; d < c.doc1; ++d) {
        w.seek(d, lane);
        const int32_t len = w.length(d);
        const int32_t src = (int32_t)w.source(d);
        for (int32_t r = 0; r < len; r += TR, ++tg) {
          const int h8 = ((len - r < TR ? len - r : TR) + 7) >> 3;  // box height / 8
          const uint32_t kbytes = (uint32_t)h8 * 1024u, S = kbytes * (uint32_t)p.kblocks;
          if (off + S > C) {  // the tile would cross the ring's end: it starts over at 0
            vpos += C - off;
            off = 0;
          }
          // tiles are consumed in order: wait for the oldest ones until none overlaps [vpos, vpos + S)
          // (tile j overlaps iff its start is less than a ring length behind this tile's end)
          while (tail < tg) {
            const uint64_t vt = __shfl_sync(0xffffffffu, vs, (int)(tail % DT_SLOTS));
            if (tg - tail < DT_SLOTS && vt + C >= vpos + S) break;
            ptx::mbar_wait(&empty[tail % DT_SLOTS], (tail / DT_SLOTS) & 1u);
            ++tail;
          }
          const uint32_t slot = tg % DT_SLOTS;
          if (lane == (int)slot) vs = vpos;
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&full[slot], S);
            for (int kb = 0; kb < p.kblocks; ++kb)
              ptx::tma_load_2d_hint(ring + off + kb * kbytes, &tm.d[h8 - 1], &full[slot], kb * 64, src + r, pol);
          }
          off += S;
          vpos += S;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (lane 0 issues; every lane runs the stream)
    uint32_t qphase = 0, tg = 0, off = 0;
    ChunkCursor cur;
    cur.init(p);
    ChunkInfo c;
    const uint32_t q_addr = ptx::smem_u32(q_slot);
    const uint32_t ring_addr = ptx::smem_u32(ring);
    const uint64_t ad0 = ptx::smem_desc_sw128(q_addr);
    const uint64_t bd_ring = ptx::smem_desc_sw128(ring_addr);  // start-address field advances by off >> 4
    const uint32_t idesc0 = p.idesc & ~(0x3Fu << 17);  // N field cleared
    while (cur.next(p, c)) {
      ptx::mbar_wait(qfull, qphase);
      ptx::tc_fence_after();
      qphase ^= 1;
      DocWindow w;
      w.open(p, c.doc0, c.doc1, lane, false);
      for (int64_t d = c.doc0; d < c.doc1; ++d) {
        w.seek(d, lane);
        const int32_t len = w.length(d);
        for (int32_t r = 0; r < len; r += TR, ++tg) {
          const int32_t h = len - r < TR ? len - r : TR;
          const uint32_t kbytes = (uint32_t)((h + 7) >> 3) * 1024u, S = kbytes * (uint32_t)p.kblocks;
          if (off + S > C) off = 0;  // the producer's placement rule
          const uint32_t idesc = idesc0 | ((uint32_t)(((h + 15) >> 4) * 2) << 17);
          const uint32_t acc = tg & accmask, slot = tg % DT_SLOTS;
          if (tg >= nacc) ptx::mbar_wait(&tempty[(tg - nacc) & 3], ((tg - nacc) >> 2) & 1);  // accumulator drained
          ptx::mbar_wait(&full[slot], (tg / DT_SLOTS) & 1u);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t d_tmem = tmem_base + acc * (uint32_t)TR;
            const uint64_t bd0 = bd_ring + (uint64_t)(off >> 4);
            const uint32_t bstep = kbytes >> 4;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
              if (kb >= p.kblocks) break;
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
                ptx::tc_mma_f16(d_tmem, ad0 + (uint64_t)(kb * 1024 + k4 * 2), bd0 + (uint64_t)(kb * bstep + k4 * 2),
                                idesc, (kb | k4) != 0);
            }
            ptx::tc_commit(&empty[slot]);
            ptx::tc_commit(&tfull[tg & 3]);
          }
          __syncwarp();
          off += S;
        }
      }
      if (lane == 0) ptx::tc_commit(qempty);
      __syncwarp();
    }
  } else if (warp >= TC_EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    // group g (nq warps, one per 32 query tokens) takes the tiles with index % rep == g; the lane of query
    // token t keeps the max over the tile's columns, merges the carry of the document's earlier tiles and,
    // on the document's last tile, the group sums over the query tokens.
    const int quad = warp - TC_EPI_WARP0;
    const int nq = p.nq, rep = p.rep;
    const int grp = quad / nq, wig = quad - grp * nq;
    if (grp < rep) {
      const float init = p.clamp_negative ? 0.0f : -INFINITY;
      const uint32_t tmem_lane = (uint32_t)(quad * 32) << 16;
      uint32_t tg = 0, pb = 0;
      ChunkCursor cursor;
      cursor.init(p);
      ChunkInfo c;
      while (cursor.next(p, c)) {
        const bool lane_valid = wig * 32 + lane < c.lq;
        DocWindow w;
        w.open(p, c.doc0, c.doc1, lane, false);
        for (int64_t d = c.doc0; d < c.doc1; ++d) {
          w.seek(d, lane);
          const int32_t len = w.length(d);
          for (int32_t r = 0; r < len; r += TR, ++tg) {
            if ((int)(tg % (uint32_t)rep) != grp) continue;
            const int ncols = len - r < TR ? len - r : TR;
            const uint32_t acc = tg & accmask;
            ptx::mbar_wait(&tfull[tg & 3], (tg >> 2) & 1);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + tmem_lane + acc * (uint32_t)TR;
            float cur = init;
            for (int c0 = 0; c0 < ncols; c0 += 128) {  // 128 columns at a time (the registers' worth)
              float v[4][32];
#pragma unroll
              for (int b = 0; b < 4; ++b)
                if (c0 + b * 32 < ncols) ptx::tmem_ld_32x32b_x32(taddr + c0 + b * 32, v[b]);
              ptx::tmem_ld_wait();
              if (c0 + 128 >= ncols) {  // the accumulator is read out: hand it back before the arithmetic
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tempty[tg & 3]);
              }
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int left = ncols - c0 - b * 32;
                if (left <= 0) break;
                if (left >= 32) cur = fmaxf(cur, max32(v[b]));
                else cur = masked_max(v[b], 0, left, cur);
              }
            }
            // carry chain (every tile waits for its predecessor's publication: keeps slot reuse ordered)
            float p_prev = init;
            if (tg > 0) {
              const uint32_t ps = (tg - 1) & 3;
              ptx::mbar_wait(&cfull[ps], ((tg - 1) >> 2) & 1);
              p_prev = carry[(ps * 4 + wig) * 32 + lane];
            }
            if (r > 0) cur = fmaxf(cur, p_prev);
            carry[((tg & 3) * 4 + wig) * 32 + lane] = cur;
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&cfull[tg & 3]);
            if (r + TR >= len) {  // the document's last tile
              const float x = warp_sum(lane_valid ? cur : 0.0f);
              if (nq == 1) {
                if (lane == 0) p.scores[d] = x;
              } else {
                if (lane == 0) part[pb * 4 + quad] = x;
                asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(nq * 32) : "memory");
                if (wig == 0 && lane == 0) {
                  float sacc = part[pb * 4 + grp * nq];
                  for (int k = 1; k < nq; ++k) sacc += part[pb * 4 + grp * nq + k];
                  p.scores[d] = sacc;
                }
                pb ^= 1;
              }
            }
          }
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
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

int make_tmap(CUtensorMap* m, const void* base, int dtype, int64_t rows, int32_t dim, uint32_t box_rows) {
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

// Interleaved view of rows [r0, r0 + 8 * groups) of a [rows, dim] token matrix (dim % 64 == 0):
// {64 cols, 8 rows, dim / 64 K blocks, groups}, one box = box_rows rows x every K block, landing in
// shared memory as box_rows / 8 groups of (dim / 64) swizzled 1 KB blocks.
static int make_tmap_ilv(CUtensorMap* m, const void* base, int dtype, int64_t r0, int64_t groups, int32_t dim,
                         uint32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(CBX_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const int32_t kb = dim / 64;
  const uint8_t* p0 = static_cast<const uint8_t*>(base) + (size_t)r0 * dim * 2;
  cuuint64_t dims[4] = {64, 8, (cuuint64_t)kb, (cuuint64_t)(groups > 0 ? groups : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)dim * 2, 128, (cuuint64_t)dim * 16};
  cuuint32_t box[4] = {64, 8, (cuuint32_t)kb, box_rows / 8};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, dtype == CBX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                   const_cast<uint8_t*>(p0), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(CBX_ECUDA, "cuTensorMapEncodeTiled (interleaved) failed (code " + std::to_string((int)r) + ")");
  return CBX_OK;
}

bool tc_supported(const cbx_batch* b) {
  return (b->dtype == CBX_F16 || b->dtype == CBX_BF16) && b->max_lq >= 1 && b->max_lq <= 128 && b->dim % 8 == 0 &&
         b->dim <= 512 && b->n_d_tokens < (int64_t(1) << 31) && b->n_q_tokens < (int64_t(1) << 31);
}

// Packed-mode plan: for candidate j (corpus document cand[j]): src_row[j], doc_len[j] and the packed
// start pk[j] = sum_{i<j} ceil8(len_i) (pk[n] = total). Three-kernel scan (block sums, their scan, add).
constexpr int PL_THREADS = 512;
constexpr int PL_PER = 8;
constexpr int PL_CHUNK = PL_THREADS * PL_PER;

__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t* wsum, int64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < PL_THREADS / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < PL_THREADS / 32) wsum[lane] = w;
  }
  __syncthreads();
  total = wsum[PL_THREADS / 32 - 1];
  const int64_t r = inc - x + (warp ? wsum[warp - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(PL_THREADS)
    plan_local_kernel(const int64_t* __restrict__ corpus_off, int64_t n_corpus, const int64_t* __restrict__ cand,
                      int64_t n, int64_t* __restrict__ pk, int64_t* __restrict__ src_row, int32_t* __restrict__ len,
                      int64_t* __restrict__ block_tot, int* __restrict__ status, int64_t pack) {
  __shared__ int64_t wsum[PL_THREADS / 32];
  const int64_t j0 = (int64_t)blockIdx.x * PL_CHUNK + (int64_t)threadIdx.x * PL_PER;
  int64_t l8[PL_PER], t = 0;
#pragma unroll
  for (int u = 0; u < PL_PER; ++u) {
    l8[u] = 0;
    const int64_t j = j0 + u;
    if (j < n) {
      const int64_t id = cand[j];
      int64_t L = 0, s0 = 0;
      if (id < 0 || id >= n_corpus) atomicOr(status, 1);
      else {
        s0 = corpus_off[id];
        L = corpus_off[id + 1] - s0;
      }
      src_row[j] = s0;
      len[j] = (int32_t)L;
      l8[u] = (L + pack - 1) & ~(pack - 1);
    }
    t += l8[u];
  }
  int64_t tot;
  int64_t run = block_excl_scan(t, wsum, tot);
#pragma unroll
  for (int u = 0; u < PL_PER; ++u) {
    if (j0 + u < n) pk[j0 + u] = run;
    run += l8[u];
  }
  if (threadIdx.x == 0) block_tot[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(PL_THREADS) plan_blocks_kernel(int64_t* __restrict__ block_tot, int64_t nb) {
  __shared__ int64_t wsum[PL_THREADS / 32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += PL_THREADS) {
    const int64_t i = base + threadIdx.x;
    const int64_t x = i < nb ? block_tot[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(x, wsum, tot);
    if (i < nb) block_tot[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) block_tot[nb] = carry;
}

__global__ void __launch_bounds__(PL_THREADS)
    plan_add_kernel(int64_t* __restrict__ pk, int64_t n, const int64_t* __restrict__ block_tot, int64_t nb) {
  const int64_t j0 = (int64_t)blockIdx.x * PL_CHUNK + (int64_t)threadIdx.x * PL_PER;
  const int64_t add = block_tot[blockIdx.x];
#pragma unroll
  for (int u = 0; u < PL_PER; ++u)
    if (j0 + u < n) pk[j0 + u] += add;
  if (blockIdx.x == 0 && threadIdx.x == 0) pk[n] = block_tot[nb];
}

size_t packed_plan_bytes(int64_t n_cand) {
  const int64_t nb = (n_cand + PL_CHUNK - 1) / PL_CHUNK;
  return align_up(8 * (size_t)(n_cand + 1), 256) + align_up(8 * (size_t)n_cand, 256) +
         align_up(4 * (size_t)n_cand, 256) + align_up(8 * (size_t)(nb + 1), 256) + 256;
}

struct TcLaunch {
  TmapSet tm;
  TcParams p;
  size_t smem;
  int grid;
};

static int prepare_tc(const cbx_batch* b, const void* d_rows, int64_t n_rows, float* scores, TcLaunch& L,
                      int tile_cap = CBX_TC_TILE256 ? 256 : 128) {
  const int kblocks = (b->dim + 63) / 64;
  // d <= 128: N = 256 MMAs (64 KB stages at d = 128); d <= 256: N = 128; d = 512: 32 rows (smem)
  int tile_n = kblocks <= 2 ? 256 : (kblocks <= 4 ? 128 : 32);
  if (tile_n > tile_cap) tile_n = tile_cap;
  const int nq = (b->max_lq + 31) / 32;
  const int rep = nq == 3 ? 1 : 4 / nq;
  const int lqp = nq * 32;
  const uint32_t q_slot_bytes = (uint32_t)(kblocks * 128 * 128);
  const uint32_t stage_bytes = (uint32_t)(kblocks * tile_n * 128);
  const size_t bar_bytes = 512 + (4 * 4 * 32 + 2 * 4 * TC_MAX_TILE_N) * sizeof(float) +
                           2 * 2 * TC_MAX_TILE_N * sizeof(int64_t);
  const size_t budget = 227 * 1024 - 1024 /*align slack*/ - bar_bytes - q_slot_bytes;
  int stages = (int)std::min<size_t>(TC_MAX_STAGES, budget / stage_bytes);
  if (stages < 2) return fail(CBX_EINVAL, "tcgen05 scorer: query tile too large for shared memory");
  L.smem = 1024 + (size_t)q_slot_bytes + (size_t)stages * stage_bytes + bar_bytes;
  for (int k = 0; k < 5; ++k) {
    const int h = tile_n >> k;
    int rc = make_tmap(&L.tm.d[k], d_rows, b->dtype, n_rows, b->dim, (uint32_t)(h >= 8 ? h : 8));
    if (rc) return rc;
  }
  int rc = make_tmap(&L.tm.q, b->q_tokens, b->dtype, b->n_q_tokens, b->dim, (uint32_t)lqp);
  if (rc) return rc;
  TcParams& p = L.p;
  p.q_tok_off = b->q_tok_off;
  p.d_tok_off = b->d_tok_off;
  p.q_doc_off = b->q_doc_off;
  p.scores = scores;
  p.packed = 0;
  p.src_row = nullptr;
  p.doc_len = nullptr;
  p.n_tokens_dev = nullptr;
  p.ilv = 0;
  p.k8 = std::min(4, 31 - __builtin_clz((unsigned)(tile_n / 8)));  // d[k8] = 8-row boxes (packed mode: tile_n <= 128)
  p.corpus_rows = n_rows;
  p.n_queries = b->n_queries;
  p.n_docs = b->n_docs;
  p.n_tokens = b->n_d_tokens;
  p.idesc = ptx::idesc_f16(b->dtype == CBX_BF16, 128, (uint32_t)tile_n);
  p.tile_n = tile_n;
  p.kblocks = kblocks;
  p.lqp = lqp;
  p.nq = nq;
  p.rep = rep;
  p.stages = stages;
  p.clamp_negative = b->clamp_negative;
  p.q_slot_bytes = q_slot_bytes;
  p.stage_bytes = stage_bytes;
  L.grid = (int)std::max<int64_t>(1, std::min<int64_t>(b->n_docs, sm_count()));
  return CBX_OK;
}

static int run_tc(const TcLaunch& L, cudaStream_t stream) {
  CBX_CUDA_CHECK(cudaFuncSetAttribute(maxsim_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
  maxsim_tc_kernel<<<L.grid, TC_THREADS, L.smem, stream>>>(L.tm, L.p);
  CBX_LAUNCH_CHECK("maxsim_tc_kernel launch");
  return CBX_OK;
}

int launch_maxsim_tc(const cbx_batch* b, float* scores, cudaStream_t stream) {
  if (!tc_supported(b)) return fail(CBX_EINVAL, "tcgen05 scorer needs f16/bf16 tokens, Lq <= 128, dim % 8 == 0");
  if (b->n_docs == 0 || b->n_queries == 0) return CBX_OK;
  TcLaunch L;
  int rc = prepare_tc(b, b->d_tokens, b->n_d_tokens, scores, L);
  if (rc) return rc;
  return run_tc(L, stream);
}

// Candidates of an HBM-resident corpus scored in place: b->d_tokens / n_d_tokens describe the corpus,
// b->q_doc_off the per-query candidate ranges of cand_ids; no copy of the candidates is made.
#ifndef CBX_PK_DOCS
#define CBX_PK_DOCS 1  // resident-corpus scoring through maxsim_docs_kernel (0: the packed tile stream, A/B knob)
#endif
int launch_maxsim_tc_packed(const cbx_batch* b, const int64_t* corpus_off, int64_t n_corpus,
                            const int64_t* cand_ids, float* scores, void* ws, size_t ws_bytes, int* status,
                            cudaStream_t stream) {
  if (!tc_supported(b)) return fail(CBX_EINVAL, "tcgen05 scorer needs f16/bf16 tokens, Lq <= 128, dim % 8 == 0");
  const int64_t n = b->n_docs;
  if (n == 0 || b->n_queries == 0) return CBX_OK;
  // document tiles of 128 rows need the K blocks of one stage to fit the ring (d <= 256)
  const bool docs = CBX_PK_DOCS && b->dim <= 256;
  if (ws_bytes < packed_plan_bytes(n)) return fail(CBX_EINVAL, "packed scorer: workspace too small");
  uint8_t* w = static_cast<uint8_t*>(ws);
  int64_t* pk = reinterpret_cast<int64_t*>(w);
  w += align_up(8 * (size_t)(n + 1), 256);
  int64_t* src = reinterpret_cast<int64_t*>(w);
  w += align_up(8 * (size_t)n, 256);
  int32_t* len = reinterpret_cast<int32_t*>(w);
  w += align_up(4 * (size_t)n, 256);
  int64_t* btot = reinterpret_cast<int64_t*>(w);
  const int64_t nb = (n + PL_CHUNK - 1) / PL_CHUNK;
  plan_local_kernel<<<(unsigned)nb, PL_THREADS, 0, stream>>>(corpus_off, n_corpus, cand_ids, n, pk, src, len, btot,
                                                             status, docs ? 8 : TC_PACK);
  CBX_LAUNCH_CHECK("plan_local_kernel launch");
  plan_blocks_kernel<<<1, PL_THREADS, 0, stream>>>(btot, nb);
  CBX_LAUNCH_CHECK("plan_blocks_kernel launch");
  plan_add_kernel<<<(unsigned)nb, PL_THREADS, 0, stream>>>(pk, n, btot, nb);
  CBX_LAUNCH_CHECK("plan_add_kernel launch");
  TcLaunch L;
  int rc = prepare_tc(b, b->d_tokens, b->n_d_tokens, scores, L, docs ? 128 : CBX_PK_TILE_N);
  if (rc) return rc;
  L.p.packed = 1;
  if (docs) {
    // one tile = up to TR rows of one document; CTAs own balanced ranges of the ceil8(len) prefix
    const int TR = L.p.kblocks <= 2 ? 256 : 128;  // a tile's K blocks must leave the ring room for several tiles
    DocTmaps tm;
    for (int h = 1; h <= DT_MAX_ROWS / 8; ++h) {
      rc = make_tmap(&tm.d[h - 1], b->d_tokens, b->dtype, b->n_d_tokens, b->dim, (uint32_t)(8 * h));
      if (rc) return rc;
    }
    tm.q = L.tm.q;
    {
      // one byte ring instead of fixed stages: everything the barrier block and the query operand leave
      const size_t bar_bytes = 512 + (4 * 4 * 32 + 8) * sizeof(float);
      const size_t ring = (227 * 1024 - 1024 /*align slack*/ - bar_bytes - L.p.q_slot_bytes - 1024 /*over-read*/) &
                          ~size_t(1023);
      L.p.stages = 1;
      L.p.stage_bytes = (uint32_t)ring;
      L.p.tile_n = TR;
      L.smem = 1024 + (size_t)L.p.q_slot_bytes + ring + 1024 + bar_bytes;
    }
    L.p.d_tok_off = pk;
    L.p.src_row = src;
    L.p.doc_len = len;
    L.p.n_tokens_dev = pk + n;
    CBX_CUDA_CHECK(cudaFuncSetAttribute(maxsim_docs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
    maxsim_docs_kernel<<<L.grid, TC_THREADS, L.smem, stream>>>(tm, L.p);
    CBX_LAUNCH_CHECK("maxsim_docs_kernel launch");
    return CBX_OK;
  }
  if (b->dim % 64 == 0) {
    for (int k = 0; k < 3; ++k) {
      const int h = L.p.tile_n >> k;
      if (h < TC_PACK) break;
      for (int r = 0; r < 8; ++r) {
        rc = make_tmap_ilv(&L.tm.pk[k][r], b->d_tokens, b->dtype, r, (b->n_d_tokens - r) / 8, b->dim, (uint32_t)h);
        if (rc) return rc;
      }
    }
    L.p.ilv = 1;
  }
  L.p.d_tok_off = pk;
  L.p.src_row = src;
  L.p.doc_len = len;
  L.p.n_tokens_dev = pk + n;
  return run_tc(L, stream);
}

}  // namespace cbx
