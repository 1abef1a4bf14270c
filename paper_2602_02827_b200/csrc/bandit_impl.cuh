// K2 — the Col-Bandit adaptive Top-K loop, one CTA per run, no host round trips.
//
// Replaces colbandit/bandit.py:169-350 (run) together with the ledger and
// reveal (oracle.py:243-329), the interval arithmetic (bounds.py:97-263) and
// numpy's Generator(PCG64) draws. Trace parity with the reference needs:
//   * float64 cells from exact products (fp16/bf16 sums are exact in fp64),
//   * CPython math.fsum semantics for every exactly rounded sum: an exact
//     int64 fixed-point accumulator (scale 2^48) while every revealed value is
//     a multiple of 2^-48 (always true for fp16 token inputs), otherwise a
//     Shewchuk expansion (Expansion) — both round correctly, like fsum,
//   * no FMA contraction and Python's left-to-right evaluation order in the
//     bound arithmetic (this translation unit is built with -fmad=false and
//     spells every operation with an explicit _rn intrinsic),
//   * numpy's PCG64 stream: next32 half-word buffering, Lemire bounded draws
//     with no draw for n == 1, random() = (next64 >> 11) * 2^-53,
//   * the loop's control flow: lazy warm-up counted as an iteration, the
//     exhausted-boundary-row switch, ties to the lower row index.
//
// Per-iteration latency chain (one CTA, 256 threads): scan the pool for the
// four boundary selections (warp redux) -> warp 0 picks i*, t* (PCG64) ->
// G-lane groups dot the document's tokens with q_t* (all loads in flight,
// float64 accumulate) -> thread 0 updates the row (Welford, exact sum,
// interval from precomputed sqrt tables) and the Top-K membership.
// Ranking and per-row state live in shared memory when the pool fits,
// otherwise in global memory.
#pragma once
#include <cstring>

#include "common.cuh"
#include "ptx.cuh"

namespace cbx {

constexpr int BD_THREADS = 256;
constexpr int BD_WARPS = BD_THREADS / 32;
constexpr int BD_CAP = 8;              // exact-sum expansion capacity (CPython fsum partials)
constexpr int BD_SMEM_ROWS = 2560;     // pools up to this size keep all per-row state in shared memory
constexpr int BD_MAX_T = 128;          // query tokens per run (the paper's queries reach 100 tokens)
constexpr double BD_FX_SCALE = 281474976710656.0;        // 2^48
constexpr double BD_FX_INV = 1.0 / 281474976710656.0;    // 2^-48
constexpr double BD_FX_LIMIT = 36028797018963968.0;      // 2^55: 128 terms stay below 2^62

static_assert(sizeof(cbx_bandit_run_desc) == 152, "cbx_bandit_run_desc layout");
static_assert(sizeof(cbx_bandit_out) == 24, "cbx_bandit_out layout");
static_assert(BD_MAX_T == CBX_BANDIT_MAX_COLS, "column capacity");

// Persistent exact-sum expansion in global memory.
struct ExpStore {
  double p[BD_CAP];
  int32_t n, pad;
};

// The unrevealed columns of a row (up to BD_MAX_T = 128), as two 64-bit words.
struct ColMask {
  uint64_t lo, hi;
  __device__ __forceinline__ bool any() const { return (lo | hi) != 0ull; }
  __device__ __forceinline__ int count() const { return __popcll(lo) + __popcll(hi); }
  __device__ __forceinline__ bool test(int t) const { return ((t < 64 ? lo >> t : hi >> (t - 64)) & 1ull) != 0ull; }
  // lowest set column
  __device__ __forceinline__ int first() const { return lo ? __ffsll((long long)lo) - 1 : 63 + __ffsll((long long)hi); }
  // the set column of rank `pos` in ascending order (pos < count())
  __device__ __forceinline__ int nth(uint32_t pos) const {
    const uint32_t c = (uint32_t)__popcll(lo);
    uint64_t m = pos < c ? lo : hi;
    const uint32_t p = pos < c ? pos : pos - c;
    for (uint32_t q = 0; q < p; ++q) m &= m - 1;  // drop the lowest p set bits
    return (pos < c ? -1 : 63) + __ffsll((long long)m);
  }
};

// Per-row state, structure of arrays: shared memory for small pools, global otherwise.
struct RowsView {
  double* proxy;
  double* lcb;
  double* ucb;
  double* mean;        // Welford running mean (oracle.py:307-310)
  double* m2;          // Welford sum of squared deviations
  long long* fx;       // exact sum of revealed values x 2^48 while every value is on that grid
  uint64_t* unrev_lo;  // bit t set = column t (< 64) not yet revealed
  uint64_t* unrev_hi;  // columns 64..127
  int32_t* cnt;        // revealed cells per row
  uint8_t* exp_mode;   // 1: the row's exact sum lives in the global expansion store
  uint8_t* member;     // Top-K membership
  __device__ void carve(uint8_t* base, int N) {
    proxy = reinterpret_cast<double*>(base);
    lcb = proxy + N;
    ucb = lcb + N;
    mean = ucb + N;
    m2 = mean + N;
    fx = reinterpret_cast<long long*>(m2 + N);
    unrev_lo = reinterpret_cast<uint64_t*>(fx + N);
    unrev_hi = unrev_lo + N;
    cnt = reinterpret_cast<int32_t*>(unrev_hi + N);
    exp_mode = reinterpret_cast<uint8_t*>(cnt + N);
    member = exp_mode + N;
  }
  __device__ __forceinline__ ColMask unrev(int i) const { return ColMask{unrev_lo[i], unrev_hi[i]}; }
};
constexpr size_t ROW_BYTES = 8 * 8 + 4 + 1 + 1;
// tournament-tree nodes get 4 bytes per row (+ CBX_BANDIT_ROW_SLACK rows of slack per run)
constexpr size_t ROW_STRIDE = ROW_BYTES + 4;
constexpr int BD_ROW_SLACK = 64;
static_assert(BD_ROW_SLACK == CBX_BANDIT_ROW_SLACK, "row slack");

struct BanditParams {
  // token source (nullptr q_tokens -> matrix source)
  const void* q_tokens;
  const int64_t* q_tok_off;
  const void* d_tokens;
  const int64_t* d_tok_off;
  int dim;
  int clamp_negative;
  const double* matrix;
  int64_t ld_matrix;
  float xmax;          // cbx_batch.d_norm_max: bound on the document tokens' norms (16-bit screen)
  int mean_doc_rows;   // n_d_tokens / n_docs of the batch (picks the wide launch shape)
  const cbx_bandit_run_desc* runs;
  const double* bounds_lo;
  const double* bounds_hi;
  const int32_t* warm_cells;
  ExpStore* g_obs;     // [rows] exact sums of rows that left the 2^-48 grid
  ExpStore* g_lo;      // [rows] sum of lo over unrevealed columns (per-cell bounds only)
  ExpStore* g_hi;      // [rows]
  uint8_t* g_rows;     // [rows * ROW_BYTES] per-row state when it does not fit in smem
  int use_smem;
  int trees_smem;      // rows global, selection trees in shared memory (set by the host when they fit)
  int bounds_smem;     // expansions (+ per-cell bounds) in shared memory at byte offset bounds_smem_off
  int64_t bounds_smem_off;
  int64_t dto_smem_off;  // > 0: the run's document offsets (n_rows + 1 int64) are staged in shared memory there
  // row-cache variant (cbx_bandit_set_row_cache; reported separately): the first adaptive reveal
  // of a row computes all of its cells from one gather (what the reference's oracle does on first touch,
  // oracle.py:210-215) and later reveals of the row read them back
  double* cell_cache;    // [trace slots] float64 cells, row-major per run at the run's trace_off
  uint8_t* row_filled;   // [state rows] 1 = the row's cells are in cell_cache
  int64_t rc_smem_off;   // shared-memory table of per-warp column front-runners (3 x 16 warps x rc_cols words)
  int32_t rc_cols;       // table columns (the launch's widest query rounded up to 8)
  int32_t rc_min_count;  // cells a row must already have revealed before a reveal fills it (default 2)
  int32_t* topk;
  int32_t max_k;
  int32_t* trace_i;
  int32_t* trace_t;
  double* trace_v;
  cbx_bandit_out* out;
  unsigned long long* prof;  // optional per-run phase cycle counters (cbx_bandit_set_profile)
  // document-sharded run (cbx_bandit_shard_step): one run, state resumed across launches
  int shard, first;
  int64_t own_lo, own_hi;   // rows whose tokens this rank holds
  int64_t* xchg;            // exchange slots, all-reduced with MAX between launches
  struct BdStep* step;
  // document-sharded run in ONE persistent launch (cbx_bandit_shard_run): the owner of a cell stores its
  // value into every peer's inbox (NVLink peer memory / this GPU's memory) and the others wait on their own
  // inbox's flag — no parking, no host round trip. CTA c of the launch is rank mb_rank0 + c.
  int mbox;
  int mb_ranks, mb_rank0;
  const cbx_mbox_peer* mb_peers;  // [grid][mb_ranks] inboxes of every rank, as seen by CTA c
  const int64_t* mb_own;          // [grid][2] owned row range of CTA c
};

// Resumable loop state of a sharded run (lives in global memory between launches).
struct BdStep {
  int32_t phase;     // CBX_SHARD_*: what the caller must exchange next
  int32_t pending;   // 0 none, 1 reveal value in xchg[0], 2 warm-up values in xchg[0..warm_m)
  int32_t status, iterations;
  int64_t n_reveals;
  int32_t i_star, t_star, swap_in, swap_out;
  int64_t warm_base, warm_m;
  uint64_t sh, sl, ih, il;
  uint32_t has32, buf;
  int32_t warmed, pad;
};
static_assert(sizeof(BdStep) <= CBX_BANDIT_STEP_BYTES, "step state");

// mailbox protocol: value store, then a release store of the flag (system scope: the inbox may be a peer
// GPU's memory over NVLink); the reader spins on an acquire load of its own inbox's flag
__device__ __forceinline__ void mbox_publish(const cbx_mbox_peer& to, int64_t slot, double v) {
  to.val[slot] = v;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(to.flag + slot), "r"(1u) : "memory");
}
__device__ __forceinline__ double mbox_wait(const cbx_mbox_peer& mine, int64_t slot) {
  uint32_t f;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(mine.flag + slot) : "memory");
  } while (f == 0u);
  return *reinterpret_cast<volatile const double*>(mine.val + slot);
}

// cell value <-> exchange slot: signed order == value order, INT64_MIN = "not mine"
__device__ __forceinline__ int64_t xchg_key(uint64_t ordkey) { return (int64_t)(ordkey ^ 0x8000000000000000ull); }
__device__ __forceinline__ uint64_t xchg_ord(int64_t k) { return (uint64_t)k ^ 0x8000000000000000ull; }

// ----------------------------------------------------------------- Python semantics
__device__ __forceinline__ double pymin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }

// ----------------------------------------------------------------- numpy PCG64
struct Pcg64 {
  uint64_t sh, sl, ih, il;
  uint32_t has32, buf;
  __device__ __forceinline__ uint64_t next64() {
    const uint64_t mh = 0x2360ED051FC65DA4ull, ml = 0x4385DF649FCCF645ull;
    uint64_t lo = sl * ml;
    uint64_t hi = __umul64hi(sl, ml) + sl * mh + sh * ml;
    uint64_t nlo = lo + il;
    hi = hi + ih + (nlo < lo ? 1ull : 0ull);
    sl = nlo;
    sh = hi;
    const uint64_t x = sh ^ sl;
    const unsigned rot = (unsigned)(sh >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf;
    }
    const uint64_t x = next64();
    has32 = 1;
    buf = (uint32_t)(x >> 32);
    return (uint32_t)x;
  }
  __device__ __forceinline__ double random() {
    return __dmul_rn((double)(next64() >> 11), 1.0 / 9007199254740992.0);
  }
  // Generator.integers(n) for 1 <= n <= 2^32 (Lemire, buffered 32-bit halves)
  __device__ __forceinline__ uint32_t integers(uint32_t n) {
    if (n <= 1) return 0;
    uint64_t m = (uint64_t)next32() * n;
    uint32_t low = (uint32_t)m;
    if (low < n) {
      const uint32_t thr = (uint32_t)((0x100000000ull - n) % n);
      while (low < thr) {
        m = (uint64_t)next32() * n;
        low = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

// ----------------------------------------------------------------- keyed selections
// order-preserving double <-> uint64
__device__ __forceinline__ uint64_t ord_key(double x) {
  uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(uint64_t k) {
  uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)u);
}

// A selection candidate: maximise `key`, break ties by minimising `tie`
// (key 0 = empty). The four selections of the loop map onto it as
//   i+      : key = ~ord(lcb),  tie = i          argmin (lcb, i) over the Top-K
//   i-      : key = ord(ucb),   tie = i          argmax ucb over the rest, lowest i
//   best    : key = ord(proxy), tie = i          first non-member in (-proxy, i)
//   worst   : key = ~ord(proxy), tie = ~i        last member in (-proxy, i)
struct Cand {
  uint64_t key;
  uint32_t tie;
};
__device__ __forceinline__ void cand_take(Cand& a, uint64_t key, uint32_t tie) {
  if (key > a.key || (key == a.key && tie < a.tie)) {
    a.key = key;
    a.tie = tie;
  }
}
// warp-wide winner: two 32-bit max reductions + one min
__device__ __forceinline__ Cand warp_best(Cand c) {
  const uint32_t hi = (uint32_t)(c.key >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t lo = hi == mh ? (uint32_t)c.key : 0u;
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lo);
  const uint64_t best = ((uint64_t)mh << 32) | ml;
  const uint32_t t = __reduce_min_sync(0xffffffffu, c.key == best ? c.tie : 0xFFFFFFFFu);
  return Cand{best, t};
}
constexpr uint32_t TIE_EMPTY = 0xFFFFFFFFu;


// ----------------------------------------------------------------- tournament trees
// Four 32-ary trees over the rows, one per selection (i+, i-, best non-member,
// worst member). Level 0 node g summarises rows [32g, 32g + 32); level l node g
// summarises level l-1 nodes [32g, 32g + 32); the single top node is the
// answer. A changed row costs one warp pass per level (32-wide redux), so a
// reveal is O(log32 N) instead of a scan of the pool.
// Level sizes and offsets are recomputed on the fly (ceil(size / 32) per level)
// so nothing here is an indexed local array: the walk stays in registers.
struct Trees {
  uint64_t* key;   // [4][nn]
  uint32_t* tie;   // [4][nn]
  int nn, nlev, size0, root_off;
  __device__ void carve(uint8_t* base, int N) {
    nlev = 0;
    nn = 0;
    size0 = (N + 31) / 32;
    int sz = size0;
    while (true) {
      root_off = nn;
      nn += sz;
      ++nlev;
      if (sz == 1 || nlev == 8) break;
      sz = (sz + 31) / 32;
    }
    key = reinterpret_cast<uint64_t*>(base);
    tie = reinterpret_cast<uint32_t*>(key + 4 * nn);
  }
  __device__ __forceinline__ Cand root(int s) const {
    const int r = s * nn + root_off;
    return Cand{key[r], tie[r]};
  }
};

// warp-collective: level-0 node g from its 32 rows (trees in `mask`: bit s = selection s)
__device__ __forceinline__ void tree_leaf(const Trees& t, const RowsView& rv, int N, int g, int lane,
                                          unsigned mask = 0xFu) {
  const int i = g * 32 + lane;
  const bool live = i < N;
  // the membership flag and the selection's value are loaded together, not one after the other: with the
  // rows in global memory (pools above BD_SMEM_ROWS) a dependent pair costs two L2 round trips per refresh
  const uint8_t memb = live ? rv.member[i] : 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (!(mask >> s & 1u)) continue;
    double val = 0.0;
    if (live) val = s == 0 ? rv.lcb[i] : (s == 1 ? rv.ucb[i] : rv.proxy[i]);
    const bool mem = memb != 0;
    // selections 0 and 3 range over members, 1 and 2 over non-members (no indexed local array)
    Cand c{0, TIE_EMPTY};
    if (live && (mem == (s == 0 || s == 3))) {
      if (s == 0) c = Cand{~ord_key(val), (uint32_t)i};
      else if (s == 1 || s == 2) c = Cand{ord_key(val), (uint32_t)i};
      else c = Cand{~ord_key(val), ~(uint32_t)i};
    }
    const Cand w = warp_best(c);
    if (lane == 0) {
      t.key[s * t.nn + g] = w.key;
      t.tie[s * t.nn + g] = w.tie;
    }
  }
}

// warp-collective: node g of a level at offset `off` from its children (level at `coff`, `csize` nodes)
__device__ __forceinline__ void tree_node(const Trees& t, int coff, int csize, int off, int g, int lane,
                                          unsigned mask = 0xFu) {
  const int c0 = g * 32 + lane;
  const bool ok = c0 < csize;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (!(mask >> s & 1u)) continue;
    Cand c{0, TIE_EMPTY};
    if (ok) {
      const int idx = s * t.nn + coff + c0;
      c = Cand{t.key[idx], t.tie[idx]};
    }
    const Cand w = warp_best(c);
    if (lane == 0) {
      t.key[s * t.nn + off + g] = w.key;
      t.tie[s * t.nn + off + g] = w.tie;
    }
  }
}

// warp-collective: refresh the path of row i in the trees of `mask`
__device__ __forceinline__ void tree_update_row(const Trees& t, const RowsView& rv, int N, int i, int lane,
                                                unsigned mask) {
  int g = i / 32;
  tree_leaf(t, rv, N, g, lane, mask);
  int coff = 0, csize = t.size0;
  for (int l = 1; l < t.nlev; ++l) {
    __syncwarp();
    g /= 32;
    const int off = coff + csize;
    tree_node(t, coff, csize, off, g, lane, mask);
    coff = off;
    csize = (csize + 31) / 32;
  }
  __syncwarp();
}

// ----------------------------------------------------------------- row arithmetic
// refresh(i) of bandit.py:220-247 / compute_decision_state (bounds.py:244-256);
// sq_log[n] = sqrt(2 log_term / n) and sq_rho[n] = sqrt(rho_n) come from tables
// built with the same operations (bounds.py:105-109, 158).
__device__ __forceinline__ void row_interval(int n, double m2, double obs, double lo_sum, double hi_sum, int T,
                                             double alpha, const double* sq_log, const double* sq_rho,
                                             double& proxy, double& lcb, double& ucb) {
  const double h_lo = __dadd_rn(obs, lo_sum);
  const double h_hi = __dadd_rn(obs, hi_sum);
  if (n == 0) {
    proxy = __dmul_rn(0.5, __dadd_rn(h_lo, h_hi));
    lcb = h_lo;
    ucb = h_hi;
    return;
  }
  const double est = (n == T) ? obs : __dmul_rn((double)T, __ddiv_rn(obs, (double)n));
  proxy = est;
  if (n <= 1) {
    lcb = h_lo;
    ucb = h_hi;
    return;
  }
  const double sigma = __dsqrt_rn(__ddiv_rn(pymax(m2, 0.0), (double)(n - 1)));
  double r = __dmul_rn(alpha, (double)T);
  r = __dmul_rn(r, sigma);
  r = __dmul_rn(r, sq_log[n]);
  r = __dmul_rn(r, sq_rho[n]);
  lcb = pymin(pymax(h_lo, __dsub_rn(est, r)), h_hi);
  ucb = pymax(pymin(h_hi, __dadd_rn(est, r)), h_lo);
}

__device__ __forceinline__ void load_exp(Expansion<BD_CAP>& e, const ExpStore& s) {
#pragma unroll
  for (int k = 0; k < BD_CAP; ++k) e.p[k] = s.p[k];
  e.n = s.n;
}
__device__ __forceinline__ void store_exp(ExpStore& s, const Expansion<BD_CAP>& e) {
#pragma unroll
  for (int k = 0; k < BD_CAP; ++k) s.p[k] = e.p[k];
  s.n = e.n;
}

// v on the 2^-48 grid with |v * 2^48| <= 2^55 -> exact int64 (sums of <= 64 stay exact)
__device__ __forceinline__ bool to_fixed(double v, long long& q) {
  const double x = __dmul_rn(v, BD_FX_SCALE);
  if (!(fabs(x) <= BD_FX_LIMIT) || x != rint(x)) return false;
  q = __double2ll_rn(x);
  return true;
}

// Slow exact-sum paths (rows whose values left the 2^-48 grid, per-cell bounds) are kept out of
// line so their 8-partial expansions do not inflate the register budget of the hot loop.
static __device__ __noinline__ bool exp_leave_grid(ExpStore* st, long long f, double v) {
  const double hi = __ll2double_rn(f);
  const double lo = __ll2double_rn(f - __double2ll_rn(hi));
  Expansion<BD_CAP> e;
  e.clear();
  bool ok = e.add(__dmul_rn(lo, BD_FX_INV));
  ok &= e.add(__dmul_rn(hi, BD_FX_INV));
  ok &= e.add(v);
  store_exp(*st, e);
  return ok;
}
// A store with n == -1 holds an exact int64 fixed-point sum (x 2^48) in p[0]: exp_init picks it when every
// value lies on the 2^-48 grid (per-cell bounds derived from fp16 tokens always do), and then a bound update
// is an integer add and one correctly rounded conversion instead of an expansion pass.
__device__ __forceinline__ double fixed_value(long long f) { return __dmul_rn(__ll2double_rn(f), BD_FX_INV); }
static __device__ __noinline__ bool exp_add(ExpStore* st, double v, double* rounded) {
  if (st->n == -1) {
    long long q;
    const long long f = __double_as_longlong(st->p[0]);
    if (to_fixed(v, q)) {
      st->p[0] = __longlong_as_double(f + q);
      if (rounded) *rounded = fixed_value(f + q);
      return true;
    }
    // off the grid after all: continue as an expansion (exact two-term split of the integer sum)
    const double hi = __ll2double_rn(f);
    const double lo = __ll2double_rn(f - __double2ll_rn(hi));
    Expansion<BD_CAP> e;
    e.clear();
    bool ok = e.add(__dmul_rn(lo, BD_FX_INV));
    ok &= e.add(__dmul_rn(hi, BD_FX_INV));
    ok &= e.add(v);
    store_exp(*st, e);
    if (rounded) *rounded = e.round();
    return ok;
  }
  Expansion<BD_CAP> e;
  load_exp(e, *st);
  const bool ok = e.add(v);
  store_exp(*st, e);
  if (rounded) *rounded = e.round();
  return ok;
}
static __device__ __noinline__ double exp_value(const ExpStore* st) {
  Expansion<BD_CAP> e;
  load_exp(e, *st);
  return e.round();
}
static __device__ __noinline__ bool exp_init(ExpStore* st, const double* vals, int n, double* rounded) {
  long long f = 0;
  bool grid = true;
  for (int t = 0; t < n && grid; ++t) {
    long long q;
    grid = to_fixed(vals[t], q);
    f += q;
  }
  if (grid) {
    st->p[0] = __longlong_as_double(f);
    st->n = -1;
    *rounded = fixed_value(f);
    return true;
  }
  Expansion<BD_CAP> e;
  e.clear();
  bool ok = true;
  for (int t = 0; t < n; ++t) ok &= e.add(vals[t]);
  store_exp(*st, e);
  *rounded = e.round();
  return ok;
}

// ----------------------------------------------------------------- cell source
// 16-byte vector of token elements -> float64 dot with a float64 slice
template <typename T>
__device__ __forceinline__ double vec_dot(const uint4& v, const double* q) {
  constexpr int PER = 16 / sizeof(T);
  const T* x = reinterpret_cast<const T*>(&v);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < PER; ++k) acc = fma(Elem<T>::to_d(x[k]), q[k], acc);
  return acc;
}

// Dot products of a range of document tokens with one query token, spread
// over `G`-lane groups: lane `sub` of a group owns 16-byte vectors
// sub, sub+G, ... of every token row (VPL of them), keeps the matching query
// slice in registers, and the group sums with log2(G) shuffles. Tokens are
// processed B at a time with every load issued before any arithmetic. Group
// `gid` handles tokens j0 + gid + k * ngroups; the trip count is kept
// warp-uniform (every lane of a warp runs the shuffles together).
template <typename T, int G, int VPL, int B>
__device__ __forceinline__ double tokens_max_dot(const T* __restrict__ dtok, int64_t j0, int64_t j1, const T* q,
                                                 int dim, int gid, int ngroups, int sub, double init) {
  constexpr int PER = 16 / sizeof(T);
  constexpr int GPW = 32 / G;  // groups per warp
  const int nvec = dim / PER;
  double qs[VPL][PER];
#pragma unroll
  for (int u = 0; u < VPL; ++u) {
    const int v = sub + u * G;
    if (v < nvec) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(q) + v);
      const T* x = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int k = 0; k < PER; ++k) qs[u][k] = Elem<T>::to_d(x[k]);
    } else {
#pragma unroll
      for (int k = 0; k < PER; ++k) qs[u][k] = 0.0;
    }
  }
  double best = init;
  const int gw = gid - gid % GPW;  // first group of this warp
  for (int64_t jw = j0 + gw; jw < j1; jw += (int64_t)ngroups * B) {
    const int64_t jb = jw + gid % GPW;
    uint4 buf[B][VPL];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int64_t j = jb + (int64_t)b * ngroups;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int v = sub + u * G;
        if (j < j1 && v < nvec) buf[b][u] = __ldg(reinterpret_cast<const uint4*>(dtok + j * dim) + v);
        else buf[b][u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < VPL; ++u) acc += vec_dot<T>(buf[b][u], qs[u]);
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const int64_t j = jb + (int64_t)b * ngroups;
      if (j < j1) best = acc > best ? acc : best;
    }
  }
  return best;
}

// 16-bit inputs: the same maximum, found by an fp32 interval screen so that
// the conversion (F2F.F64, 16 lanes per clock per SM) and float64 shuffle
// work of the MIO pipe — which bound the all-float64 scan above — is spent
// on one or two rows per warp instead of every row.
//  * Layout: SG lanes per token row, each owning SV = 4 16-byte vectors
//    (sub, sub + SG, ...): log2(SG) fp32 butterfly levels per row (SG = 4 for
//    d = 128 16-bit tokens, against 4 float64 levels in tokens_max_dot).
//  * Interval: a product of two fp16 (11-bit) or bf16 (8-bit) significands is
//    exact in fp32, so the fp32 dot s of a row is within
//    gamma_36 * sum|x_k q_k| <= 2^-18.8 |x| |q| of its float64 value
//    (Cauchy-Schwarz; <= 37 roundings per lane chain + butterfly). With
//    eps = 2^-16 xmax |q| + 2^-40, xmax = cbx_batch.d_norm_max >= |x| for
//    every document token (|q|^2 accumulated in fp32; 2^-40 absorbs bf16
//    products and squares that underflow), the row's value lies in
//    [lb, ub] = [s - eps, s + eps], rounded outwards: one radius for the whole
//    reveal, so rows carry no norms (a third fewer FMAs and half the shuffles
//    of a per-row |x|). Queries with |q|^2 outside [2^-60, 2^60] are not
//    screened (every row is exact).
//  * Prune: LB = max(clamp floor, best exact value, every lb seen) is a lower
//    bound on the answer, so a row with ub < LB cannot be (or tie) the
//    maximum. Rows with ub >= LB wait in a per-warp list (entry k in lane k)
//    and are recomputed in float64 by the whole warp — highest ub first, one
//    16-byte vector per lane, fma chain + butterfly — when the list fills or
//    the range ends; each exact value raises LB and prunes the rest. NaN or
//    overflowed intervals are never pruned and never raise LB.
// The result is the exact maximum of the float64 dots, as in tokens_max_dot.
__device__ __forceinline__ uint32_t ord_key_f(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <typename T, int SG, int B>
__device__ __forceinline__ double tokens_max_screen(const T* __restrict__ dtok, int64_t j0, int64_t j1,
                                                    const T* __restrict__ q, int dim, int wid, int nwarps, int lane,
                                                    double best, const unsigned long long* shared_best, float xmax) {
  constexpr int SV = 4;
  constexpr int RPW = 32 / SG;
  constexpr int EV = (SG * SV + 31) / 32;
  const int nvec = dim / 8;
  const int sub = lane % SG, grp = lane / SG;
  float qf[SV][8];
  float nq2 = 0.0f;
#pragma unroll
  for (int u = 0; u < SV; ++u) {
    const int v = sub + u * SG;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (v < nvec) w = __ldg(reinterpret_cast<const uint4*>(q) + v);
    const T* x = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      qf[u][k] = Elem<T>::to_f(x[k]);
      nq2 = __fmaf_rn(qf[u][k], qf[u][k], nq2);
    }
  }
#pragma unroll
  for (int o = SG / 2; o > 0; o >>= 1) nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, o));
  const bool screen = nq2 >= 0x1p-60f && nq2 <= 0x1p60f && xmax <= 0x1p60f;
  const float qn = __fsqrt_ru(nq2);
  // one error radius for every row: |x| <= xmax (cbx_batch.d_norm_max) bounds the fp32 rounding error of any
  // row's dot by 2^-18.8 xmax |q| (Cauchy-Schwarz), so the rows need no norms of their own
  const float eps = __fmaf_ru(__fmul_ru(xmax, qn), 0x1p-16f, 0x1p-40f);
  float LB = best == -INFINITY ? -INFINITY : __double2float_rd(best);
  float p_ub = -INFINITY;  // pending list: entry `lane`
  int64_t p_j = 0;
  int pc = 0;

  // exact float64 value of pending rows, highest ub first, until none can reach LB
  auto flush = [&]() {
    while (true) {
      const uint32_t key = (lane < pc && !(p_ub < LB)) ? ord_key_f(p_ub) | 1u : 0u;  // NaN ub: ord_key_f > 0
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
      if (kmax == 0u) break;
      const int L = __ffs(__ballot_sync(0xffffffffu, key == kmax)) - 1;
      const int64_t j = __shfl_sync(0xffffffffu, p_j, L);
      if (lane == L) p_ub = -INFINITY;
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        const int v = lane + 32 * e;
        if (v < nvec) {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(dtok + j * dim) + v);
          const uint4 qw = __ldg(reinterpret_cast<const uint4*>(q) + v);
          const T* x = reinterpret_cast<const T*>(&w);
          const T* y = reinterpret_cast<const T*>(&qw);
          double part = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) part = fma(Elem<T>::to_d(x[k]), Elem<T>::to_d(y[k]), part);
          acc += part;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (acc > best) {
        best = acc;
        LB = fmaxf(LB, __double2float_rd(acc));
      }
    }
    pc = 0;
  };

  const int64_t ngroups = (int64_t)nwarps * RPW;
  for (int64_t jw = j0 + (int64_t)wid * RPW; jw < j1; jw += ngroups * B) {  // warp-uniform
    uint4 buf[B][SV];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int64_t j = jw + grp + (int64_t)b * ngroups;
#pragma unroll
      for (int u = 0; u < SV; ++u) {
        const int v = sub + u * SG;
        if (j < j1 && v < nvec) buf[b][u] = __ldg(reinterpret_cast<const uint4*>(dtok + j * dim) + v);
        else buf[b][u] = make_uint4(0, 0, 0, 0);
      }
    }
    float ub[B];
    float lbmax = -INFINITY;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float s = 0.0f;
#pragma unroll
      for (int u = 0; u < SV; ++u) {
        const T* x = reinterpret_cast<const T*>(&buf[b][u]);
#pragma unroll
        for (int k = 0; k < 8; ++k) s = __fmaf_rn(Elem<T>::to_f(x[k]), qf[u][k], s);
      }
#pragma unroll
      for (int o = SG / 2; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      const int64_t j = jw + grp + (int64_t)b * ngroups;
      const bool live = j < j1;
      ub[b] = !live ? -INFINITY : (screen ? __fadd_ru(s, eps) : INFINITY);
      const float lb = __fsub_rd(s, eps);
      if (live && screen && lb <= 3.0e38f && lb >= -3.0e38f) lbmax = fmaxf(lbmax, lb);  // finite only
    }
    if (shared_best) {
      const double sb = ord_val(*reinterpret_cast<const volatile unsigned long long*>(shared_best));
      if (sb > best) best = sb;
    }
    // LB over the warp: the largest finite lb of this step (ordered-key max), the best exact value
    const uint32_t lk = __reduce_max_sync(0xffffffffu, lbmax == -INFINITY ? 0u : ord_key_f(lbmax));
    if (lk) LB = fmaxf(LB, __uint_as_float((lk & 0x80000000u) ? (lk & 0x7FFFFFFFu) : ~lk));
    if (best != -INFINITY) LB = fmaxf(LB, __double2float_rd(best));
#pragma unroll
    for (int b = 0; b < B; ++b) {
      unsigned m = __ballot_sync(0xffffffffu, sub == 0 && !(ub[b] < LB));
      while (m) {  // warp-uniform: append the row of group leader L to the pending list
        const int L = __ffs(m) - 1;
        m &= m - 1;
        const float u = __shfl_sync(0xffffffffu, ub[b], L);
        if (lane == pc) {
          p_ub = u;
          p_j = jw + L / SG + (int64_t)b * ngroups;
        }
        if (++pc == 32) flush();
      }
    }
  }
  if (shared_best) {
    const double sb = ord_val(*reinterpret_cast<const volatile unsigned long long*>(shared_best));
    if (sb > best) {
      best = sb;
      LB = fmaxf(LB, __double2float_rd(sb));
    }
  }
  flush();
  return best;
}

// 16-bit inputs with dim <= 256: the same interval screen with the fp32 dots taken by the
// warp-level tensor-core MMA (mma.sync m16n8k16, fp32 accumulate) straight from registers — the reveal is a
// latency-bound GEMV over one document, so operands staged through shared memory (TMA + tcgen05) would add a
// barrier round trip per document, while the FMA screen above spends ~250 issue slots per 16 rows and warp;
// this one spends ~25 (8 LDG.128 + 8 HMMA per 16 rows at d = 128).
//  * A = 16 document tokens x 16 k per instruction. Lane (g = lane / 4, t = lane % 4) loads the 16-byte
//    vector t of every 64-byte chunk of rows g and g + 8 (each warp load covers whole 32-byte sectors) and
//    feeds its four words as the fragment's k positions {2t, 2t+1, 2t+8, 2t+9}: a dot product does not care
//    about the order of k as long as B uses the same one, so B's fragment is the query's vector at the same
//    byte offset. The query sits in every one of B's 8 columns: each lane reads its rows' sums off c0 / c2.
//  * eps = dim 2^-19 xmax |q| + 2^-40 bounds the accumulation error of the tensor core's fp32 adder (exact
//    16-bit products; the bound Stage 1 uses for tcgen05, validated there against the float64 scan).
//  * LB is shared by the CTA's warps through an ordered-key atomicMax in shared memory (`shared_lb`) and a
//    barrier before the exact pass, so only rows within 2 eps of the document's best fp32 dot — one or two
//    per reveal — are recomputed in float64, straight from the registers that still hold them (no second
//    load) and in the fma / summation order of the FMA screen's exact pass (row_dot_exact), bit for bit.
template <typename T>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __half>::value)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ord_val_f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
// Variant A (default, CBX_BD_MMA_REGS = 0): rows that survive the screen wait in a per-warp list and are
// re-read (L1 / L2 hits) for the exact pass — the 64 staging registers are dead once the MMAs have consumed
// them. Variant B (CBX_BD_MMA_REGS = 1, tokens_max_mma below) takes the exact dots from the staging registers
// themselves; inside this kernel it spills (ptxas: 600 B of stack at the 128-register cap the two-CTA-per-SM
// occupancy imposes) and measured 2x slower, so it is kept as a build knob only.
template <typename T, int KCMAX, int BT>
__device__ __forceinline__ double tokens_max_mma_reload(const T* __restrict__ dtok, int64_t j0, int64_t j1,
                                                 const T* __restrict__ q, int dim, int wid, int nwarps, int lane,
                                                 double best, unsigned int* shared_lb, float xmax) {
  const int nvec = dim >> 3;        // 16-byte vectors per row
  const int kc = (nvec + 3) >> 2;   // 64-byte chunks per row (the last one zero-padded when dim % 32 != 0)
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntile = (j1 - j0 + 15) >> 4;
  const int64_t stride = (int64_t)nwarps * BT;
  uint4 U[BT][KCMAX], V[BT][KCMAX];
  // one step's loads: rows g and g + 8 of BT tiles (issued before anything that waits on data)
  auto load_step = [&](int64_t tb) {
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
      const uint4* p0 = reinterpret_cast<const uint4*>(dtok + r0 * dim) + t;
      const uint4* p1 = reinterpret_cast<const uint4*>(dtok + (r0 + 8) * dim) + t;
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        U[b][c] = make_uint4(0, 0, 0, 0);
        V[b][c] = make_uint4(0, 0, 0, 0);
        if (c * 4 + t < nvec && r0 < j1) U[b][c] = __ldg(p0 + c * 4);
        if (c * 4 + t < nvec && r0 + 8 < j1) V[b][c] = __ldg(p1 + c * 4);
      }
    }
  };
  uint4 qv[KCMAX];
#pragma unroll
  for (int c = 0; c < KCMAX; ++c) {
    qv[c] = make_uint4(0, 0, 0, 0);
    if (c * 4 + t < nvec) qv[c] = __ldg(reinterpret_cast<const uint4*>(q) + c * 4 + t);
  }
  float nq2 = 0.0f;
#pragma unroll
  for (int c = 0; c < KCMAX; ++c) {
    const T* x = reinterpret_cast<const T*>(&qv[c]);
#pragma unroll
    for (int k = 0; k < 8; ++k) nq2 = __fmaf_rn(Elem<T>::to_f(x[k]), Elem<T>::to_f(x[k]), nq2);
  }
  nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, 1));
  nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, 2));
  const bool screen = nq2 >= 0x1p-60f && nq2 <= 0x1p60f && xmax <= 0x1p60f;
  const float qn = __fmul_ru(__fsqrt_ru(nq2), 1.0000005f);  // the fp32 |q|^2 above is within 2^-20 of the exact one
  const float eps = __fmaf_ru(__fmul_ru(__fmul_ru(xmax, qn), (float)dim), 0x1p-19f, 0x1p-40f);
  float LB = best == -INFINITY ? -INFINITY : __double2float_rd(best);
  float p_ub = -INFINITY;  // pending list: entry `lane`
  int64_t p_j = 0;
  int pc = 0;

  // exact float64 value of pending rows, highest ub first, until none can reach LB
  auto flush = [&]() {
    while (true) {
      const uint32_t key = (lane < pc && !(p_ub < LB)) ? ord_key_f(p_ub) | 1u : 0u;  // NaN ub: ord_key_f > 0
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
      if (kmax == 0u) break;
      const int L = __ffs(__ballot_sync(0xffffffffu, key == kmax)) - 1;
      const int64_t j = __shfl_sync(0xffffffffu, p_j, L);
      if (lane == L) p_ub = -INFINITY;
      double acc = 0.0;
      if (lane < nvec) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(dtok + j * dim) + lane);
        const uint4 qw = __ldg(reinterpret_cast<const uint4*>(q) + lane);
        const T* x = reinterpret_cast<const T*>(&w);
        const T* y = reinterpret_cast<const T*>(&qw);
        double part = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) part = fma(Elem<T>::to_d(x[k]), Elem<T>::to_d(y[k]), part);
        acc += part;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (acc > best) {
        best = acc;
        LB = fmaxf(LB, __double2float_rd(acc));
      }
    }
    pc = 0;
  };

  for (int64_t tb = wid; tb < ntile; tb += stride) {  // warp-uniform
    load_step(tb);
    float sv[BT][2];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        if (c < kc) {
          mma16816<T>(acc, U[b][c].x, V[b][c].x, U[b][c].y, V[b][c].y, qv[c].x, qv[c].y);
          mma16816<T>(acc, U[b][c].z, V[b][c].z, U[b][c].w, V[b][c].w, qv[c].z, qv[c].w);
        }
      }
      sv[b][0] = acc[0];
      sv[b][1] = acc[2];
    }
    float ub[BT][2];
    float lbmax = -INFINITY;
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float s = sv[b][h];
        const bool live = r0 + 8 * h < j1;
        ub[b][h] = !live ? -INFINITY : (screen ? __fadd_ru(s, eps) : INFINITY);
        const float lb = __fsub_rd(s, eps);
        if (live && screen && lb <= 3.0e38f && lb >= -3.0e38f) lbmax = fmaxf(lbmax, lb);  // finite only
      }
    }
    // LB over the warp (and, through shared_lb, over the CTA's warps so far)
    const uint32_t lk = __reduce_max_sync(0xffffffffu, lbmax == -INFINITY ? 0u : ord_key_f(lbmax));
    if (lk) LB = fmaxf(LB, ord_val_f(lk));
    if (shared_lb) {
      if (lane == 0 && lk) atomicMax(shared_lb, lk);
      const uint32_t sk = *reinterpret_cast<volatile unsigned int*>(shared_lb);
      if (sk) LB = fmaxf(LB, ord_val_f(sk));
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        unsigned m = __ballot_sync(0xffffffffu, t == 0 && !(ub[b][h] < LB));
        while (m) {  // warp-uniform: append the row of lane L to the pending list
          const int L = __ffs(m) - 1;
          m &= m - 1;
          const float u = __shfl_sync(0xffffffffu, ub[b][h], L);
          if (lane == pc) {
            p_ub = u;
            p_j = j0 + ((tb + (int64_t)b * nwarps) << 4) + (L >> 2) + 8 * h;
          }
          if (++pc == 32) flush();
        }
      }
    }
  }
  if (shared_lb) {
    // every warp has published its rows' lower bounds: the exact pass only sees the document's front-runners
    __syncthreads();
    const uint32_t sk = *reinterpret_cast<volatile unsigned int*>(shared_lb);
    if (sk) LB = fmaxf(LB, ord_val_f(sk));
  }
  flush();
  return best;
}

#ifndef CBX_BD_STREAM_NOALLOC
#define CBX_BD_STREAM_NOALLOC 1  // document tokens bypass L1 allocation (read once per reveal; L1 keeps the run's metadata)
#endif
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
#if CBX_BD_STREAM_NOALLOC
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
// float64 dot of the 8 + 8 elements of two 16-byte vectors, k ascending from +0.0 (the exact pass's chain)
template <typename T>
__device__ __forceinline__ double vec_dot_exact(const uint4& w, const uint4& qw) {
  const T* x = reinterpret_cast<const T*>(&w);
  const T* y = reinterpret_cast<const T*>(&qw);
  double part = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) part = fma(Elem<T>::to_d(x[k]), Elem<T>::to_d(y[k]), part);
  return part;
}
// The exact float64 dot of a row held as KCMAX vectors per lane (vector index v = 4 c + t over the row's four
// lanes t), summed in exactly the order of the one-vector-per-lane butterfly used everywhere else in this
// file (xor 16, 8, 4, 2, 1 over v): the xor 16 / 8 / 4 levels pair vectors of the same lane (c ^ 4, c ^ 2,
// c ^ 1; absent vectors are +0.0, as idle lanes are there), xor 2 and 1 are shuffles between the four lanes.
template <typename T, int KCMAX>
__device__ __forceinline__ double row_dot_exact(const uint4 (&r)[KCMAX], const uint4 (&qv)[KCMAX]) {
  double P[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) P[c] = 0.0;
#pragma unroll
  for (int c = 0; c < KCMAX; ++c) P[c] = vec_dot_exact<T>(r[c], qv[c]);
  double s;
  if constexpr (KCMAX > 4) {
    const double q0 = P[0] + P[4], q1 = P[1] + P[5], q2 = P[2] + P[6], q3 = P[3] + P[7];  // xor 16
    s = (q0 + q2) + (q1 + q3);                                                           // xor 8, xor 4
  } else if constexpr (KCMAX > 2) {
    s = (P[0] + P[2]) + (P[1] + P[3]);  // xor 8, xor 4
  } else if constexpr (KCMAX > 1) {
    s = P[0] + P[1];  // xor 4
  } else {
    s = P[0];
  }
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}
#ifndef CBX_BD_MMA_NOINLINE
#define CBX_BD_MMA_NOINLINE 0  // 1: the register variant as a real call (measured no better: the call is merged back)
#endif
#if CBX_BD_MMA_NOINLINE
#define CBX_BD_MMA_LINKAGE static __device__ __noinline__
#else
#define CBX_BD_MMA_LINKAGE __device__ __forceinline__
#endif
template <typename T, int KCMAX, int BT>
CBX_BD_MMA_LINKAGE double tokens_max_mma(const T* __restrict__ dtok, int64_t j0, int64_t j1,
                                                 const T* __restrict__ q, int dim, int wid, int nwarps, int lane,
                                                 double best, unsigned int* shared_lb, float xmax) {
  const int nvec = dim >> 3;        // 16-byte vectors per row
  const int kc = (nvec + 3) >> 2;   // 64-byte chunks per row (the last one zero-padded when dim % 32 != 0)
  const int g = lane >> 2, t = lane & 3;
  const int64_t ntile = (j1 - j0 + 15) >> 4;
  const int64_t stride = (int64_t)nwarps * BT;
  uint4 U[BT][KCMAX], V[BT][KCMAX];
  // one step's loads: rows g and g + 8 of BT tiles (issued before anything that waits on data)
  auto load_step = [&](int64_t tb) {
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
      const uint4* p0 = reinterpret_cast<const uint4*>(dtok + r0 * dim) + t;
      const uint4* p1 = reinterpret_cast<const uint4*>(dtok + (r0 + 8) * dim) + t;
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        U[b][c] = make_uint4(0, 0, 0, 0);
        V[b][c] = make_uint4(0, 0, 0, 0);
        if (c * 4 + t < nvec && r0 < j1) U[b][c] = ld_stream(p0 + c * 4);
        if (c * 4 + t < nvec && r0 + 8 < j1) V[b][c] = ld_stream(p1 + c * 4);
      }
    }
  };
  uint4 qv[KCMAX];
#pragma unroll
  for (int c = 0; c < KCMAX; ++c) {
    qv[c] = make_uint4(0, 0, 0, 0);
    if (c * 4 + t < nvec) qv[c] = __ldg(reinterpret_cast<const uint4*>(q) + c * 4 + t);
  }
  const bool have = wid < ntile;
  if (have) load_step(wid);  // the document's first rows are in flight while |q| is taken
  float nq2 = 0.0f;
#pragma unroll
  for (int c = 0; c < KCMAX; ++c) {
    const T* x = reinterpret_cast<const T*>(&qv[c]);
#pragma unroll
    for (int k = 0; k < 8; ++k) nq2 = __fmaf_rn(Elem<T>::to_f(x[k]), Elem<T>::to_f(x[k]), nq2);
  }
  nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, 1));
  nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, 2));
  const bool screen = nq2 >= 0x1p-60f && nq2 <= 0x1p60f && xmax <= 0x1p60f;
  const float qn = __fmul_ru(__fsqrt_ru(nq2), 1.0000005f);  // the fp32 |q|^2 above is within 2^-20 of the exact one
  const float eps = __fmaf_ru(__fmul_ru(__fmul_ru(xmax, qn), (float)dim), 0x1p-19f, 0x1p-40f);
  float LB = best == -INFINITY ? -INFINITY : __double2float_rd(best);
  float ub[BT][2];

  // rows that may hold the maximum (ub >= LB): their exact float64 dots, taken from the registers that hold
  // the rows — all eight rows of a (tile, half) at once, one per lane group
  auto resolve = [&]() {
#pragma unroll
    for (int b = 0; b < BT; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!__any_sync(0xffffffffu, !(ub[b][h] < LB))) continue;  // warp-uniform
        const double e = h ? row_dot_exact<T, KCMAX>(V[b], qv) : row_dot_exact<T, KCMAX>(U[b], qv);
        // max over the live rows (a dead row's ub is -inf; non-candidates cannot exceed the maximum anyway)
        const uint64_t k = ub[b][h] == -INFINITY ? 0ull : ord_key(e);
        const uint32_t kh = (uint32_t)(k >> 32);
        const uint32_t mh = __reduce_max_sync(0xffffffffu, kh);
        const uint32_t ml = __reduce_max_sync(0xffffffffu, kh == mh ? (uint32_t)k : 0u);
        const uint64_t km = ((uint64_t)mh << 32) | ml;
        if (km) {
          const double m = ord_val(km);
          if (m > best) {
            best = m;
            LB = fmaxf(LB, __double2float_rd(m));
          }
        }
      }
    }
  };

  int64_t tb = wid;
  bool pending = false;  // the last step's rows wait for the CTA-wide bound
  while (have) {  // warp-uniform
    float lbmax = -INFINITY;
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        if (c < kc) {
          mma16816<T>(acc, U[b][c].x, V[b][c].x, U[b][c].y, V[b][c].y, qv[c].x, qv[c].y);
          mma16816<T>(acc, U[b][c].z, V[b][c].z, U[b][c].w, V[b][c].w, qv[c].z, qv[c].w);
        }
      }
      const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float s = h ? acc[2] : acc[0];
        const bool live = r0 + 8 * h < j1;
        ub[b][h] = !live ? -INFINITY : (screen ? __fadd_ru(s, eps) : INFINITY);
        const float lb = __fsub_rd(s, eps);
        if (live && screen && lb <= 3.0e38f && lb >= -3.0e38f) lbmax = fmaxf(lbmax, lb);  // finite only
      }
    }
    // LB over the warp (and, through shared_lb, over the CTA's warps so far)
    const uint32_t lk = __reduce_max_sync(0xffffffffu, lbmax == -INFINITY ? 0u : ord_key_f(lbmax));
    if (lk) LB = fmaxf(LB, ord_val_f(lk));
    if (shared_lb) {
      if (lane == 0 && lk) atomicMax(shared_lb, lk);
      const uint32_t sk = *reinterpret_cast<volatile unsigned int*>(shared_lb);
      if (sk) LB = fmaxf(LB, ord_val_f(sk));
    }
    if (tb + stride >= ntile) {
      pending = true;
      break;
    }
    resolve();  // before the registers take the next step's rows
    tb += stride;
    load_step(tb);
  }
  if (shared_lb) {
    // every warp has published its rows' lower bounds: the exact pass only sees the document's front-runners
    __syncthreads();
    const uint32_t sk = *reinterpret_cast<volatile unsigned int*>(shared_lb);
    if (sk) LB = fmaxf(LB, ord_val_f(sk));
  }
  if (pending) resolve();
  return best;
}

// Row-cache variant: ALL cells H[i, 0..TC) of one document from one gather. Same tensor-core screen as
// tokens_max_mma_reload, but B carries 8 different query tokens per pass (TC / 8 passes over the staged
// rows), so a lane reads two columns of two rows per tile off its C fragment. Each warp keeps, per column,
// the largest and second-largest fp32 dot of its rows and the row of the largest (shared-memory table, one
// slot per warp and column); after one barrier, column n is resolved by warp n % nwarps: every warp's
// front-runner within 2 eps of the best is recomputed in float64 (re-read, same fma / butterfly order as
// everywhere else), and if any warp's SECOND row could also reach the bound — or anything was not finite —
// the column falls back to the exact single-column scan. The cells are the exact maxima either way.
template <typename T, int KCMAX, int BT>
__device__ __forceinline__ void row_cells_mma(const T* __restrict__ dtok, int64_t j0, int64_t j1,
                                              const T* __restrict__ qtok, int TC, int dim, int wid, int nwarps,
                                              int lane, double init, float xmax, float* tab, int TCP,
                                              double* __restrict__ out_cells, int t_star,
                                              unsigned long long* cellkey) {
  const int nvec = dim >> 3;
  const int kc = (nvec + 3) >> 2;
  const int g = lane >> 2, t = lane & 3;
  float* cmax1 = tab + (size_t)wid * TCP;
  float* cmax2 = tab + (size_t)(16 + wid) * TCP;
  int* crow = reinterpret_cast<int*>(tab + (size_t)(32 + wid) * TCP);
  for (int n = lane; n < TCP; n += 32) {
    cmax1[n] = -INFINITY;
    cmax2[n] = -INFINITY;
    crow[n] = -1;
  }
  __syncwarp();
  const int64_t ntile = (j1 - j0 + 15) >> 4;
  const int64_t stride = (int64_t)nwarps * BT;
  for (int64_t tb = wid; tb < ntile; tb += stride) {  // warp-uniform
    uint4 U[BT][KCMAX], V[BT][KCMAX];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
      const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
      const uint4* p0 = reinterpret_cast<const uint4*>(dtok + r0 * dim) + t;
      const uint4* p1 = reinterpret_cast<const uint4*>(dtok + (r0 + 8) * dim) + t;
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        U[b][c] = make_uint4(0, 0, 0, 0);
        V[b][c] = make_uint4(0, 0, 0, 0);
        if (c * 4 + t < nvec && r0 < j1) U[b][c] = __ldg(p0 + c * 4);
        if (c * 4 + t < nvec && r0 + 8 < j1) V[b][c] = __ldg(p1 + c * 4);
      }
    }
    for (int cb = 0; cb * 8 < TC; ++cb) {
      // B fragment: query token cb * 8 + g in column g
      uint4 qv[KCMAX];
      const int qi = cb * 8 + g;
#pragma unroll
      for (int c = 0; c < KCMAX; ++c) {
        qv[c] = make_uint4(0, 0, 0, 0);
        if (qi < TC && c * 4 + t < nvec) qv[c] = __ldg(reinterpret_cast<const uint4*>(qtok + (int64_t)qi * dim) + c * 4 + t);
      }
      // this lane's columns 2t (k = 0) and 2t + 1 (k = 1): largest, second largest, row of the largest
      float m1[2] = {-INFINITY, -INFINITY}, m2[2] = {-INFINITY, -INFINITY};
      int r1[2] = {-1, -1};
#pragma unroll
      for (int b = 0; b < BT; ++b) {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < KCMAX; ++c) {
          if (c < kc) {
            mma16816<T>(acc, U[b][c].x, V[b][c].x, U[b][c].y, V[b][c].y, qv[c].x, qv[c].y);
            mma16816<T>(acc, U[b][c].z, V[b][c].z, U[b][c].w, V[b][c].w, qv[c].z, qv[c].w);
          }
        }
        const int64_t r0 = j0 + ((tb + (int64_t)b * nwarps) << 4) + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (r0 + 8 * h < j1) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              float sv = acc[2 * h + k];
              if (!(fabsf(sv) <= 3.0e38f)) sv = INFINITY;  // NaN / overflow: forces the exact fallback below
              if (sv > m1[k]) {
                m2[k] = m1[k];
                m1[k] = sv;
                r1[k] = (int)(r0 + 8 * h - j0);
              } else if (sv > m2[k]) {
                m2[k] = sv;
              }
            }
          }
        }
      }
      // merge over the 8 row groups (lanes with the same t)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float a1 = __shfl_xor_sync(0xffffffffu, m1[k], o);
          const float a2 = __shfl_xor_sync(0xffffffffu, m2[k], o);
          const int ar = __shfl_xor_sync(0xffffffffu, r1[k], o);
          if (a1 > m1[k]) {
            m2[k] = fmaxf(m1[k], a2);
            m1[k] = a1;
            r1[k] = ar;
          } else {
            m2[k] = fmaxf(m2[k], a1);
          }
        }
      }
      if (g == 0) {  // fold into the warp's table (earlier steps of a long document)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int n = cb * 8 + 2 * t + k;
          const float o1 = cmax1[n], o2 = cmax2[n];
          if (m1[k] > o1) {
            cmax1[n] = m1[k];
            cmax2[n] = fmaxf(o1, m2[k]);
            crow[n] = r1[k];
          } else {
            cmax2[n] = fmaxf(o2, m1[k]);
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();  // every warp's front-runners are in the table
  const float* all1 = tab;
  const float* all2 = tab + (size_t)16 * TCP;
  const int* allr = reinterpret_cast<const int*>(tab + (size_t)32 * TCP);
  for (int n = wid; n < TC; n += nwarps) {  // warp-uniform
    const T* q = qtok + (int64_t)n * dim;
    uint4 qw = make_uint4(0, 0, 0, 0);
    if (lane < nvec) qw = __ldg(reinterpret_cast<const uint4*>(q) + lane);
    float nq2 = 0.0f;
    {
      const T* y = reinterpret_cast<const T*>(&qw);
#pragma unroll
      for (int k = 0; k < 8; ++k) nq2 = __fmaf_rn(Elem<T>::to_f(y[k]), Elem<T>::to_f(y[k]), nq2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nq2 = __fadd_rn(nq2, __shfl_xor_sync(0xffffffffu, nq2, o));
    const bool screen = nq2 >= 0x1p-60f && nq2 <= 0x1p60f && xmax <= 0x1p60f;
    const float qn = __fmul_ru(__fsqrt_ru(nq2), 1.0000005f);
    const float eps = __fmaf_ru(__fmul_ru(__fmul_ru(xmax, qn), (float)dim), 0x1p-19f, 0x1p-40f);
    const float w1 = lane < nwarps ? all1[(size_t)lane * TCP + n] : -INFINITY;
    const float w2 = lane < nwarps ? all2[(size_t)lane * TCP + n] : -INFINITY;
    const int wr = lane < nwarps ? allr[(size_t)lane * TCP + n] : -1;
    float top = w1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = fmaxf(top, __shfl_xor_sync(0xffffffffu, top, o));
    float LB = top == -INFINITY ? -INFINITY : __fsub_rd(top, eps);
    if (init != -INFINITY) LB = fmaxf(LB, __double2float_rd(init));
    // a second row of some warp could reach the bound, or a value was not finite: exact scan of the column
    const bool amb = !screen || top == INFINITY ||
                     __any_sync(0xffffffffu, w2 != -INFINITY && !(__fadd_ru(w2, eps) < LB));
    double v = init;
    if (amb) {
      v = tokens_max_mma_reload<T, KCMAX, BT>(dtok, j0, j1, q, dim, 0, 1, lane, init, nullptr, xmax);
    } else {
      unsigned m = __ballot_sync(0xffffffffu, wr >= 0 && !(__fadd_ru(w1, eps) < LB));
      while (m) {  // warp-uniform
        const int L = __ffs(m) - 1;
        m &= m - 1;
        const int64_t j = j0 + __shfl_sync(0xffffffffu, wr, L);
        double acc = 0.0;
        if (lane < nvec) acc = vec_dot_exact<T>(__ldg(reinterpret_cast<const uint4*>(dtok + j * dim) + lane), qw);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (acc > v) v = acc;
      }
    }
    if (lane == 0) {
      out_cells[n] = v;
      if (n == t_star) *cellkey = ord_key(v);
    }
  }
}

#ifndef CBX_BD_MMA_REGS
#define CBX_BD_MMA_REGS 0
#endif
#ifndef CBX_BD_MMA
#define CBX_BD_MMA 1  // tensor-core (mma.sync) screen for 16-bit tokens with dim <= 256
#endif
#ifndef CBX_BD_SCREEN
#define CBX_BD_SCREEN 1
#endif
#ifndef CBX_BD_SCREEN_B
#define CBX_BD_SCREEN_B 2  // rows per lane group in flight
#endif
// maximum over tokens [j0, j1) of the float64 dot with q; `init` is the clamp floor.
// (G, VPL) is the all-float64 layout; wid/nwarps/lane place the calling warp for the screened layout;
// xmax bounds the document tokens' norms (screened layout).
// WBT > 0: the calling kernel owns its SM's register file (one CTA per SM, up to 255 registers per thread):
// the tensor-core screen then stages WBT tiles per warp and step and takes the exact dots from the staging
// registers (tokens_max_mma) — no second load of the front-runner rows.
#ifndef CBX_BD_WIDE_BT
#define CBX_BD_WIDE_BT 2  // 16-row tiles staged per warp and step in wide launches (d <= 128; 3 spills at 255 registers)
#endif
#ifndef CBX_BD_WARM_BT
#define CBX_BD_WARM_BT 3  // the same in the warm-up pre-pass kernel (248 registers, no spills)
#endif
template <typename T, int G, int VPL>
__host__ __device__ constexpr bool bd_mma_layout() { return sizeof(T) == 2 && CBX_BD_SCREEN && CBX_BD_MMA && G * VPL <= 32; }
template <typename T, int G, int VPL, int B, int WBT = 0>
__device__ __forceinline__ double tokens_max(const T* __restrict__ dtok, int64_t j0, int64_t j1, const T* q, int dim,
                                             int gid, int ngroups, int sub, double init, int wid, int nwarps,
                                             const unsigned long long* shared_best, unsigned int* shared_lb, float xmax) {
  if constexpr (sizeof(T) == 2 && CBX_BD_SCREEN) {
    if constexpr (CBX_BD_MMA && G * VPL <= 32) {
      constexpr int KCMAX = (G * VPL) / 4;
      if constexpr (WBT > 0)  // WBT tiles per warp and step for d <= 128 (4 staging registers per tile and 32 dims)
        return tokens_max_mma<T, KCMAX, (KCMAX <= 4 ? WBT : (WBT + 1) / 2)>(dtok, j0, j1, q, dim, wid, nwarps,
                                                                            threadIdx.x & 31, init, shared_lb, xmax);
#if CBX_BD_MMA_REGS
      return tokens_max_mma<T, KCMAX, (KCMAX <= 4 ? 2 : 1)>(dtok, j0, j1, q, dim, wid, nwarps, threadIdx.x & 31, init,
                                                             shared_lb, xmax);
#else
      return tokens_max_mma_reload<T, KCMAX, (KCMAX <= 4 ? 2 : 1)>(dtok, j0, j1, q, dim, wid, nwarps,
                                                                    threadIdx.x & 31, init, shared_lb, xmax);
#endif
    }
    constexpr int SG = (G * VPL) / 4 < 1 ? 1 : (G * VPL) / 4;
    return tokens_max_screen<T, SG, CBX_BD_SCREEN_B>(dtok, j0, j1, q, dim, wid, nwarps, threadIdx.x & 31, init,
                                                      shared_best, xmax);
  } else {
    return tokens_max_dot<T, G, VPL, B>(dtok, j0, j1, q, dim, gid, ngroups, sub, init);
  }
}

// ----------------------------------------------------------------- the kernel
#ifndef CBX_BD_DOC_PREFETCH
#define CBX_BD_DOC_PREFETCH 1  // decision loads i*'s token range and starts an L2 bulk prefetch of the document
#endif
#ifndef CBX_BD_TRACE_WARP
#define CBX_BD_TRACE_WARP 1    // warp 1 writes the trace entry (off thread 0's critical path)
#endif
// SM: where the per-row state and the selection trees live — 2: both in shared memory (pools up to
// BD_SMEM_ROWS), 1: rows in global memory, trees in shared memory (one big run per SM), 0: both global.
// A compile-time placement lets every row/tree access be a plain LDS/STS (or LDG/STG) instead of a generic
// load: generic loads that resolve to shared memory still queue in the SM's global-memory pipeline, behind
// a co-resident CTA's reveal (measured: ~4.7k cycles of thread 0's row update per cfg2 iteration).
// threads per CTA: NT = 256 is two runs per SM (register file split, 128 registers per thread); NT = 512 is
// the "wide" launch, every run with an SM to itself, in one of two shapes: 512 threads of 128 registers
// (16 warps x 2 tiles = 512 rows per reveal step: long documents, cfg3's 1030 rows), or — WREG, tensor-core
// screen only — 256 threads of up to 255 registers, whose reveal keeps its rows in registers for the exact
// pass (8 warps x 2 tiles = 256 rows per step: documents of a few hundred rows, cfg4). The launcher picks by
// the batch's mean document length.
template <int NT, bool WREG>
__host__ __device__ constexpr int bd_threads() { return NT == 512 && WREG ? 256 : NT; }
// RC: the row-cache variant is compiled into its own instantiations (its code in the default kernel cost the
// on-demand loop ~20 % through register allocation and code placement: cfg2 11.0 -> 13.5 ms, measured)
template <typename T, int G, int VPL, int NT, bool UNI, int SM, bool WREG = false, bool RC = false>
__global__ void __launch_bounds__(bd_threads<NT, WREG>(), NT == 256 ? 2 : 1) bandit_kernel(const BanditParams P) {
  static_assert(!WREG || (NT == 512 && bd_mma_layout<T, G, VPL>()), "WREG is a wide tensor-core-screen shape");
  static_assert(!RC || (UNI && bd_mma_layout<T, G, VPL>()), "the row cache serves generic-bounds runs on the MMA layouts");
  constexpr bool WIDE = WREG;  // rows stay in the staging registers for the exact pass
  constexpr int BD_THREADS = bd_threads<NT, WREG>();
  constexpr int BD_WARPS = BD_THREADS / 32;
  extern __shared__ __align__(16) uint8_t bd_smem[];
  constexpr int NGROUPS = BD_THREADS / G;
#ifndef CBX_BD_TOKENS_IN_FLIGHT
#define CBX_BD_TOKENS_IN_FLIGHT 8
#endif
  constexpr int B = VPL == 1 ? CBX_BD_TOKENS_IN_FLIGHT : (VPL == 2 ? CBX_BD_TOKENS_IN_FLIGHT / 2 : CBX_BD_TOKENS_IN_FLIGHT / 4);
  constexpr int GW = G <= 32 ? G : 32;
  const cbx_bandit_run_desc R = P.runs[blockIdx.x];
  const int N = R.n_rows, TC = R.n_cols, K = R.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = tid / G, sub = tid % G;
  // descriptors live in device memory, so the C ABI cannot check them on the host: a run outside the
  // kernel's shape contract reports CBX_BANDIT_EDESC instead of overrunning its masks and tables
  if (N < 1 || TC < 1 || TC > BD_MAX_T || K < 1 || K > N || K > P.max_k) {
    if (tid == 0) {
      cbx_bandit_out o;
      o.n_reveals = 0;
      o.iterations = 0;
      o.terminated_by = CBX_TERM_SEPARATION;
      o.status = CBX_BANDIT_EDESC;
      o.pad = 0;
      P.out[blockIdx.x] = o;
      if (P.shard && P.step) P.step->phase = CBX_SHARD_DONE;
    }
    return;
  }
  // owned rows of this CTA's rank (sharded runs)
  const int64_t own_lo = P.mbox ? P.mb_own[2 * blockIdx.x] : P.own_lo;
  const int64_t own_hi = P.mbox ? P.mb_own[2 * blockIdx.x + 1] : P.own_hi;
  const int my_rank = P.mbox ? P.mb_rank0 + (int)blockIdx.x : 0;
  const cbx_mbox_peer* peers = P.mbox ? P.mb_peers + (size_t)blockIdx.x * P.mb_ranks : nullptr;
  // UNI: every run of the launch has uniform (generic) bounds, so the per-cell-bound code compiles away
  // (a smaller hot loop: measured 2-4 % faster on cfg2/3/5)
  const bool uniform = UNI || R.bounds_off < 0;
  const double* lo_b = uniform ? nullptr : P.bounds_lo + R.bounds_off;
  const double* hi_b = uniform ? nullptr : P.bounds_hi + R.bounds_off;
  const bool tokens = P.q_tokens != nullptr;
  const int dim = P.dim;
  // row-cache variant: token-backed runs with generic bounds on the tensor-core screen's layouts
  const bool rcache = RC && P.cell_cache != nullptr && tokens && !P.shard;

  struct Ctrl {
    int action;       // 0 reveal, 1 stop, 2 warm-up, 3 exhaustion, 4 error
    int i_star, t_star;
    int status;
    int64_t n_reveals;
    int iterations;
    unsigned int lbkey;         // CTA-wide fp32 lower bound of the cell being revealed (ordered key, 0 = none)
    unsigned long long cellkey;
    int32_t swap_in, swap_out;  // best non-member / worst member of the last selection
    int32_t partner;            // row whose membership swapped with i* this iteration (-1: none)
    int32_t hit;                // row-cache variant: the cell of this iteration came from the cache
    int32_t fills;              // row-cache variant: rows whose cells were computed (one gather each)
    int64_t j0, j1;             // token range of i* (read by the decision with its other loads)
  };
  static_assert(sizeof(Ctrl) <= 128, "control block");
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(bd_smem);
  Cand* red = reinterpret_cast<Cand*>(bd_smem + 128);                 // [4][BD_WARPS]
  double* sq_log = reinterpret_cast<double*>(red + 4 * 16);           // [BD_MAX_T + 1]
  double* sq_rho = sq_log + BD_MAX_T + 1;                             // [BD_MAX_T + 1]
  uint8_t* row_base;
  if constexpr (SM == 2) row_base = reinterpret_cast<uint8_t*>(sq_rho + BD_MAX_T + 1);
  else row_base = P.g_rows + (size_t)R.state_off * ROW_STRIDE;
  RowsView rv;
  rv.carve(row_base, N);
  const bool use_tree = (R.flags & CBX_BANDIT_TREE) != 0;
  Trees tr;
  // trees in shared memory when the rows are in global memory but the CTA has the SM to itself
  // (one run per SM: decide and the per-level tree walks become shared-memory round trips)
  if constexpr (SM == 1) tr.carve(reinterpret_cast<uint8_t*>(sq_rho + BD_MAX_T + 1), N);
  else tr.carve(row_base + align_up_dev(ROW_BYTES * (size_t)N, 16), N);
  ExpStore* g_obs = P.g_obs + R.state_off;
  ExpStore* g_lo = P.g_lo + R.state_off;
  ExpStore* g_hi = P.g_hi + R.state_off;
  if (P.bounds_smem) {
    // one run per SM and a small pool: the exact-sum expansions and the per-cell bounds are staged in
    // shared memory, so the greedy column choice and the interval updates stop paying HBM round trips
    ExpStore* se = reinterpret_cast<ExpStore*>(bd_smem + P.bounds_smem_off);
    g_obs = se;
    g_lo = se + N;
    g_hi = se + 2 * N;
    if (!uniform) {
      double* slo = reinterpret_cast<double*>(se + 3 * N);
      double* shi = slo + (size_t)N * TC;
      for (int64_t x = tid; x < (int64_t)N * TC; x += BD_THREADS) {
        slo[x] = lo_b[x];
        shi[x] = hi_b[x];
      }
      lo_b = slo;
      hi_b = shi;
    }
    __syncthreads();
  }
  int32_t* tr_i = P.trace_i + R.trace_off;
  int32_t* tr_t = P.trace_t + R.trace_off;
  double* tr_v = P.trace_v + R.trace_off;

  const T* qtok = nullptr;
  const T* dtok = nullptr;
  const int64_t* dto = nullptr;
  if (tokens) {
    qtok = static_cast<const T*>(P.q_tokens) + P.q_tok_off[R.query] * (int64_t)dim;
    dtok = static_cast<const T*>(P.d_tokens);
    dto = P.d_tok_off + R.row_begin;
  }
  const double init_cell = P.clamp_negative ? 0.0 : -INFINITY;
  // the decision reads the token ranges of both boundary rows every iteration: from shared memory when the
  // run's offsets fit there (an L2 round trip per iteration otherwise)
  const int64_t* dto_s = nullptr;
  if (SM == 2 && tokens && P.dto_smem_off > 0) {
    int64_t* d = reinterpret_cast<int64_t*>(bd_smem + P.dto_smem_off);
    for (int i = tid; i <= N; i += BD_THREADS) d[i] = dto[i];
    dto_s = d;
    __syncthreads();
  }

  // optional phase cycle counters (thread 0; cbx_bandit_set_profile)
  unsigned long long ph[16] = {0};
  unsigned long long tc0 = clock64();
#define BD_PHASE(k)                            \
  do {                                         \
    if (__builtin_expect(P.prof != nullptr, 0) && tid == 0) { \
      const unsigned long long _n = clock64(); \
      ph[k] += _n - tc0;                       \
      tc0 = _n;                                \
    }                                          \
  } while (0)
  // exact sum of a row's revealed values, rounded like math.fsum
  auto obs_sum = [&](int i) -> double {
    if (__builtin_expect(rv.exp_mode[i], 0)) return exp_value(&g_obs[i]);
    return __dmul_rn(__ll2double_rn(rv.fx[i]), BD_FX_INV);
  };
  // add v to row i's exact sum; false on expansion overflow
  auto obs_add = [&](int i, double v) -> bool {
    long long q;
    if (__builtin_expect(!rv.exp_mode[i], 1)) {
      if (__builtin_expect(to_fixed(v, q), 1)) {
        rv.fx[i] += q;
        return true;
      }
      // leave the grid: the int64 sum becomes an exact two-term expansion
      rv.exp_mode[i] = 1;
      return exp_leave_grid(&g_obs[i], rv.fx[i], v);
    }
    return exp_add(&g_obs[i], v, nullptr);
  };

  // ledger._record (oracle.py:305-314) + refresh(i) (bandit.py:220-247) for one row
  // pre: the two unrevealed-bound sums after removing column t, already computed (per-cell bounds)
  double last_proxy = 0.0;  // proxy written by the last reveal_update of this thread (saves re-reading it)
  auto reveal_update = [&](int i, int t, double v, bool have_pre = false, double pre_lo = 0.0,
                           double pre_hi = 0.0) -> bool {
    // every load of the row up front, in one batch: with the rows in global memory (pools above BD_SMEM_ROWS)
    // each read-modify-write below would otherwise stall the thread for its own L2 round trip
    const int n = rv.cnt[i] + 1;
    double mean = rv.mean[i], m2 = rv.m2[i];
    const uint8_t em = rv.exp_mode[i];
    long long fx = rv.fx[i];
    const uint64_t ulo = rv.unrev_lo[i], uhi = rv.unrev_hi[i];
    BD_PHASE(8);
    const double d = __dsub_rn(v, mean);
    mean = __dadd_rn(mean, __ddiv_rn(d, (double)n));
    m2 = __dadd_rn(m2, __dmul_rn(d, __dsub_rn(v, mean)));
    BD_PHASE(9);
    // the row's exact sum (math.fsum of its revealed values): int64 fixed point on the 2^-48 grid, else an expansion
    bool ok = true;
    double obs;
    long long q;
    if (__builtin_expect(!em, 1)) {
      if (__builtin_expect(to_fixed(v, q), 1)) {
        fx += q;
        rv.fx[i] = fx;
        obs = __dmul_rn(__ll2double_rn(fx), BD_FX_INV);
      } else {  // leave the grid: the int64 sum becomes an exact two-term expansion
        rv.exp_mode[i] = 1;
        ok = exp_leave_grid(&g_obs[i], fx, v);
        obs = exp_value(&g_obs[i]);
      }
    } else {
      ok = exp_add(&g_obs[i], v, &obs);
    }
    BD_PHASE(10);
    rv.mean[i] = mean;
    rv.m2[i] = m2;
    if (t < 64) rv.unrev_lo[i] = ulo & ~(1ull << t);
    else rv.unrev_hi[i] = uhi & ~(1ull << (t - 64));
    rv.cnt[i] = n;
    double lo_sum, hi_sum;
    if (uniform) {
      // fsum of (T - n) copies of a constant == the correctly rounded product
      lo_sum = (TC - n) ? __dmul_rn((double)(TC - n), R.lo_uniform) : 0.0;
      hi_sum = (TC - n) ? __dmul_rn((double)(TC - n), R.hi_uniform) : 0.0;
    } else if (have_pre) {
      lo_sum = pre_lo;
      hi_sum = pre_hi;
    } else {
      ok &= exp_add(&g_lo[i], -lo_b[(int64_t)i * TC + t], &lo_sum);
      ok &= exp_add(&g_hi[i], -hi_b[(int64_t)i * TC + t], &hi_sum);
    }
    double px, l, u;
    row_interval(n, m2, obs, lo_sum, hi_sum, TC, R.alpha_ef, sq_log, sq_rho, px, l, u);
    rv.proxy[i] = px;
    rv.lcb[i] = l;
    rv.ucb[i] = u;
    last_proxy = px;
    BD_PHASE(11);
    return ok;
  };

  // H[i, t] by one warp (warm-up cells)
  auto cell_warp = [&](int i, int t) -> double {
    if (!tokens) return P.matrix[(R.row_begin + i) * P.ld_matrix + t];
    double best = tokens_max<T, GW, VPL, (VPL == 1 ? 8 : 4), WIDE ? CBX_BD_WIDE_BT : 0>(dtok, dto[i], dto[i + 1],
                                                                         qtok + (int64_t)t * dim, dim, lane / GW,
                                                                         32 / GW, lane % GW, init_cell, 0, 1, nullptr,
                                                                         nullptr, P.xmax);
#pragma unroll
    for (int o = 16; o >= GW; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, best, o);
      best = w > best ? w : best;
    }
    return best;
  };

  // rebuild(): membership = first K rows of the (-proxy, i) order (bandit.py:251-263)
  auto rebuild = [&]() {
    for (int i = tid; i < N; i += BD_THREADS) rv.member[i] = 0;
    __syncthreads();
    for (int r = 0; r < K; ++r) {
      Cand c{0, TIE_EMPTY};
      for (int i = tid; i < N; i += BD_THREADS)
        if (!rv.member[i]) cand_take(c, ord_key(rv.proxy[i]), (uint32_t)i);
      c = warp_best(c);
      if (lane == 0) red[warp] = c;
      __syncthreads();
      if (warp == 0) {
        Cand b = lane < BD_WARPS ? red[lane] : Cand{0, TIE_EMPTY};
        b = warp_best(b);
        if (lane == 0) rv.member[b.tie] = 1;
      }
      __syncthreads();
    }
    if (use_tree) {
      int coff = 0, csize = tr.size0;
      for (int l = 0; l < tr.nlev; ++l) {
        const int off = l == 0 ? 0 : coff + csize;
        const int size = l == 0 ? tr.size0 : (csize + 31) / 32;
        for (int g = warp; g < size; g += BD_WARPS) {
          if (l == 0) tree_leaf(tr, rv, N, g, lane);
          else tree_node(tr, coff, csize, off, g, lane);
        }
        if (l > 0) {
          coff = off;
          csize = size;
        }
        __syncthreads();
      }
    }
  };

  // ------------------------------------------------------------ initial state (all n = 0)
  BdStep* const step = P.step;
  const bool resume = P.shard && !P.mbox && !P.first;
  if (P.shard && !P.mbox && step->phase == CBX_SHARD_DONE) return;
  if (tid == 0) {
    ctrl->status = resume ? step->status : 0;
    ctrl->n_reveals = resume ? step->n_reveals : 0;
    ctrl->iterations = resume ? step->iterations : 0;
    ctrl->fills = 0;
    ctrl->hit = 0;
    if (resume) {
      ctrl->i_star = step->i_star;
      ctrl->t_star = step->t_star;
      ctrl->swap_in = step->swap_in;
      ctrl->swap_out = step->swap_out;
    }
  }
  for (int n = tid; n <= BD_MAX_T; n += BD_THREADS) {
    double a = 0.0, b = 0.0;
    if (n >= 1 && n <= TC) {
      a = __dsqrt_rn(__ddiv_rn(__dmul_rn(2.0, R.log_term), (double)n));
      double rho;
      if (2 * n <= TC) rho = __dsub_rn(1.0, __ddiv_rn((double)(n - 1), (double)TC));
      else rho = __dmul_rn(__dsub_rn(1.0, __ddiv_rn((double)n, (double)TC)), __dadd_rn(1.0, __ddiv_rn(1.0, (double)n)));
      b = __dsqrt_rn(rho);
    }
    sq_log[n] = a;
    sq_rho[n] = b;
  }
  __syncthreads();
  const uint64_t full_lo = TC >= 64 ? ~0ull : ((1ull << TC) - 1ull);
  const uint64_t full_hi = TC >= 128 ? ~0ull : (TC <= 64 ? 0ull : ((1ull << (TC - 64)) - 1ull));
  for (int i = resume ? N : tid; i < N; i += BD_THREADS) {
    rv.mean[i] = 0.0;
    rv.m2[i] = 0.0;
    rv.fx[i] = 0;
    rv.exp_mode[i] = 0;
    rv.unrev_lo[i] = full_lo;
    rv.unrev_hi[i] = full_hi;
    rv.cnt[i] = 0;
    double lo_sum, hi_sum;
    if (uniform) {
      lo_sum = __dmul_rn((double)TC, R.lo_uniform);
      hi_sum = __dmul_rn((double)TC, R.hi_uniform);
    } else {
      bool ok = exp_init(&g_lo[i], lo_b + (int64_t)i * TC, TC, &lo_sum);
      ok &= exp_init(&g_hi[i], hi_b + (int64_t)i * TC, TC, &hi_sum);
      if (!ok) ctrl->status = 2;
    }
    double px, l, u;
    row_interval(0, 0.0, 0.0, lo_sum, hi_sum, TC, R.alpha_ef, sq_log, sq_rho, px, l, u);
    rv.proxy[i] = px;
    rv.lcb[i] = l;
    rv.ucb[i] = u;
  }
  __syncthreads();
  if (!resume) rebuild();

  Pcg64 rng;
  rng.sh = resume ? step->sh : R.rng.state_hi;
  rng.sl = resume ? step->sl : R.rng.state_lo;
  rng.ih = resume ? step->ih : R.rng.inc_hi;
  rng.il = resume ? step->il : R.rng.inc_lo;
  rng.has32 = resume ? step->has32 : R.rng.has_uint32;
  rng.buf = resume ? step->buf : R.rng.uinteger;
  bool warmed = resume ? step->warmed != 0 : ((K == N) || (R.explore_mode == CBX_UNIFORM_ROW));
  int resume_kind = resume ? step->pending : 0;
  // sharded run: park the loop at an exchange point (thread 0 holds the live generator)
  auto park = [&](int pending, int phase, int64_t wbase, int64_t wm) {
    if (tid == 0) {
      step->phase = phase;
      step->pending = pending;
      step->status = ctrl->status;
      step->iterations = ctrl->iterations;
      step->n_reveals = ctrl->n_reveals;
      step->i_star = ctrl->i_star;
      step->t_star = ctrl->t_star;
      step->swap_in = ctrl->swap_in;
      step->swap_out = ctrl->swap_out;
      step->warm_base = wbase;
      step->warm_m = wm;
      step->sh = rng.sh;
      step->sl = rng.sl;
      step->ih = rng.ih;
      step->il = rng.il;
      step->has32 = rng.has32;
      step->buf = rng.buf;
      step->warmed = warmed ? 1 : 0;
    }
  };
  // apply the m warm-up reveals recorded at trace[base, base + m) (bandit.py:285-296)
  auto warmup_apply = [&](int64_t base, int64_t m) {
    // epsilon-greedy: one cell per row (trace slot base + i holds row i), rows in parallel; static warm-up:
    // cells may share rows, so thread 0 applies them in draw order. One call site of reveal_update.
    const bool par = R.explore_mode == CBX_EPSILON_GREEDY;
    for (int64_t s2 = par ? tid : (tid == 0 ? 0 : m); s2 < m; s2 += par ? BD_THREADS : 1)
      if (!reveal_update(tr_i[base + s2], tr_t[base + s2], tr_v[base + s2])) ctrl->status = 2;
    __syncthreads();
    if (m > 0) rebuild();
    if (tid == 0) ctrl->n_reveals = base + m;
    __syncthreads();
  };
  const double eps = R.explore_mode == CBX_UNIFORM_ROW ? 1.0 : R.epsilon;
  const int64_t total_cells = (int64_t)N * TC;
  int term = CBX_TERM_SEPARATION;
  tc0 = clock64();
  const unsigned long long tcs = tc0;

  while (true) {
    BD_PHASE(3);
    int i_star, t_star;
    int64_t wa_base = 0, wa_m = -1;  // a warm-up to apply this iteration
    if (__builtin_expect(resume_kind == 0, 1)) {
    // ---------------------------------------------------------- boundary selection
    if (__builtin_expect(!use_tree, 0)) {
      Cand c[4] = {{0, TIE_EMPTY}, {0, TIE_EMPTY}, {0, TIE_EMPTY}, {0, TIE_EMPTY}};
      for (int i = tid; i < N; i += BD_THREADS) {
        const uint64_t pk = ord_key(rv.proxy[i]);
        if (rv.member[i]) {
          cand_take(c[0], ~ord_key(rv.lcb[i]), (uint32_t)i);
          cand_take(c[3], ~pk, ~(uint32_t)i);
        } else {
          cand_take(c[1], ord_key(rv.ucb[i]), (uint32_t)i);
          cand_take(c[2], pk, (uint32_t)i);
        }
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const Cand w = warp_best(c[s]);
        if (lane == 0) red[s * BD_WARPS + warp] = w;
      }
      __syncthreads();
    }
    BD_PHASE(0);
    if (warp == 0) {
      int wsel_i = -1;
      int pf_row = -1;  // the row about to be revealed (rows in global memory: its lines are prefetched below)
      ColMask wsel_un{0ull, 0ull};
      Cand f[4];
      if (use_tree) {
#pragma unroll
        for (int s = 0; s < 4; ++s) f[s] = tr.root(s);
      } else {
#pragma unroll
        for (int s = 0; s < 4; ++s)
          f[s] = warp_best(lane < BD_WARPS ? red[s * BD_WARPS + lane] : Cand{0, TIE_EMPTY});
      }
      if (lane == 0) {
        ctrl->iterations += 1;
        ctrl->swap_in = f[2].key ? (int)f[2].tie : -1;
        ctrl->swap_out = f[3].key ? (int)~f[3].tie : -1;
        const int i_plus = (int)f[0].tie;
        const int i_minus = f[1].key ? (int)f[1].tie : -1;
        const int im = i_minus >= 0 ? i_minus : i_plus;  // a valid row for the loads below
        // the selection keys carry the bounds (key 0 = ~ord(lcb) over members, key 1 = ord(ucb) over the rest)
        const double lcb_plus = ord_val(~f[0].key);
        const double ucb_minus = i_minus >= 0 ? ord_val(f[1].key) : -INFINITY;
        // everything else the decision may read, issued together (one round trip when rows live in HBM)
        const double ucb_p = rv.ucb[i_plus], lcb_m = rv.lcb[im];
        const ColMask un_p = rv.unrev(i_plus), un_m = rv.unrev(im);
#if CBX_BD_DOC_PREFETCH
        // both candidates' token ranges come with the same round trip, so the reveal does not pay one
        int64_t jp0 = 0, jp1 = 0, jm0 = 0, jm1 = 0;
        if (tokens) {
          const int64_t* o = (SM == 2 && dto_s) ? dto_s : dto;
          jp0 = o[i_plus];
          jp1 = o[i_plus + 1];
          jm0 = o[im];
          jm1 = o[im + 1];
        }
#endif
        int action;
        if (lcb_plus >= ucb_minus) {
          action = 1;
        } else if (!warmed) {
          action = 2;
          warmed = true;
        } else if (ctrl->n_reveals == total_cells) {
          action = 3;
        } else {
          action = 0;
          const double wp = __dsub_rn(ucb_p, lcb_plus);
          const double wm = __dsub_rn(ucb_minus, lcb_m);
          int i_star = wp >= wm ? i_plus : i_minus;
          ColMask un = i_star == i_plus ? un_p : un_m;
          if (!un.any()) {
            i_star = i_star == i_plus ? i_minus : i_plus;
            un = i_star == i_plus ? un_p : un_m;
            if (!un.any()) {
              action = 4;
              ctrl->status = 1;
            }
          }
          if (action == 0) {
            int t_star;
            if (rng.random() < eps) {
              t_star = un.nth(rng.integers((uint32_t)un.count()));
            } else if (uniform) {
              t_star = un.first();  // all widths equal: first unrevealed column
            } else {
              // first argmax of the width over the ascending unrevealed columns: warp 0 below
              t_star = -1;
              wsel_i = i_star;
              wsel_un = un;
            }
            ctrl->i_star = i_star;
            pf_row = i_star;
            ctrl->t_star = t_star;
            ctrl->cellkey = ord_key(init_cell);
            ctrl->lbkey = 0u;
            if constexpr (RC) {
              if (rcache) {
                // both loads at once; the cached value only counts when the row has been filled. A row is
                // filled on the reveal that finds rc_min_count cells of it already revealed: rows that never
                // get that far (most of a pool: the warm-up cell plus one adaptive reveal) stay on demand
                const uint8_t f = P.row_filled[R.state_off + i_star];
                const double cv = P.cell_cache[R.trace_off + (int64_t)i_star * TC + t_star];
                ctrl->hit = f ? 1 : (TC - un.count() >= P.rc_min_count ? 0 : 2);  // 2: on demand, no fill
                if (f) ctrl->cellkey = ord_key(cv);
              }
            }
#if CBX_BD_DOC_PREFETCH
            if (tokens) {
              const int64_t j0 = i_star == i_plus ? jp0 : jm0, j1 = i_star == i_plus ? jp1 : jm1;
              ctrl->j0 = j0;
              ctrl->j1 = j1;
              // start streaming the document into L2 now; the reveal's loads then meet it on the way
              const uint32_t nb = (uint32_t)((j1 - j0) * (int64_t)dim * (int64_t)sizeof(T));
              if (nb >= 16 && (!P.shard || (i_star >= own_lo && i_star < own_hi)) && !(RC && rcache && ctrl->hit == 1))
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(dtok + j0 * dim), "r"(nb) : "memory");
#if CBX_BD_DOC_PREFETCH >= 2
              // the other boundary row is often the next one revealed: warm it as well
              const int other = i_star == i_plus ? i_minus : i_plus;
              if (other >= 0) {
                const int64_t o0 = other == i_plus ? jp0 : jm0, o1 = other == i_plus ? jp1 : jm1;
                const uint32_t ob = (uint32_t)((o1 - o0) * (int64_t)dim * (int64_t)sizeof(T));
                if (ob >= 16 && (!P.shard || (other >= own_lo && other < own_hi)))
                  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(dtok + o0 * dim), "r"(ob) : "memory");
              }
#endif
            }
#endif
          }
        }
        ctrl->action = action;
      }
#ifndef CBX_BD_ROW_PREFETCH
#define CBX_BD_ROW_PREFETCH 0  // measured on cfg4: decide 1.9k -> 4.5k cycles, 1.79 -> 2.15 s (the prefetches queue in front of the decision); off
#endif
      if constexpr (SM != 2 && CBX_BD_ROW_PREFETCH) {
        // rows live in global memory (pools above BD_SMEM_ROWS): one lane per line pulls what the row update,
        // the membership test and the tree-leaf refresh of i* will read into L1 while the reveal runs (the
        // reveal's own token loads do not allocate in L1 in the wide register shape)
        const int pr = __shfl_sync(0xffffffffu, pf_row, 0);
        if (pr >= 0) {
          const int g0 = pr & ~31, g1 = min(g0 + 31, N - 1);
          const void* a = nullptr;
          switch (lane) {
            case 0: a = rv.cnt + pr; break;
            case 1: a = rv.mean + pr; break;
            case 2: a = rv.m2 + pr; break;
            case 3: a = rv.fx + pr; break;
            case 4: a = rv.unrev_lo + pr; break;
            case 5: a = rv.unrev_hi + pr; break;
            case 6: a = rv.exp_mode + pr; break;
            case 7: a = rv.member + g0; break;
            case 8: a = rv.lcb + g0; break;
            case 9: a = rv.lcb + g1; break;
            case 10: a = rv.ucb + g0; break;
            case 11: a = rv.ucb + g1; break;
            case 12: a = rv.proxy + g0; break;
            case 13: a = rv.proxy + g1; break;
            default: break;
          }
          if (a) asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
        }
      }
      const int wi = uniform ? -1 : __shfl_sync(0xffffffffu, wsel_i, 0);
      if (wi >= 0) {  // one column per lane, warp argmax, ties to the lowest column (select_token, bandit.py:116-136)
        const ColMask un{__shfl_sync(0xffffffffu, wsel_un.lo, 0), __shfl_sync(0xffffffffu, wsel_un.hi, 0)};
        Cand c{0, TIE_EMPTY};
        for (int t = lane; t < TC; t += 32)
          if (un.test(t))
            cand_take(c, ord_key(__dsub_rn(hi_b[(int64_t)wi * TC + t], lo_b[(int64_t)wi * TC + t])), (uint32_t)t);
        c = warp_best(c);
        if (lane == 0) ctrl->t_star = c.key ? (int)c.tie : un.first();
      }
    }
    __syncthreads();
    BD_PHASE(1);
    const int action = ctrl->action;
    if (action == 1) break;
    if (action == 3) {
      term = CBX_TERM_EXHAUSTION;
      break;
    }
    if (action == 4) break;

    if (__builtin_expect(action == 2, 0)) {
      // -------------------------------------------------------- lazy warm-up (bandit.py:285-296)
      warmed = true;
      const int64_t base = ctrl->n_reveals;
      const int64_t m = R.explore_mode == CBX_EPSILON_GREEDY ? N : R.n_warm;
      // cells computed by cbx_bandit_prewarm already sit in trace[0, m) (the warm-up is the first reveal)
      const bool pre = (R.flags & CBX_BANDIT_PREWARMED) && base == 0 && !P.shard;
      if (R.explore_mode == CBX_EPSILON_GREEDY) {
        if (tid == 0)
          for (int i = 0; i < N; ++i) {
            const int32_t t = (int32_t)rng.integers((uint32_t)TC);
            if (!pre) {
              tr_i[base + i] = i;
              tr_t[base + i] = t;
            }
          }
      } else if (!pre) {
        const int32_t* wc = P.warm_cells + R.warm_off;
        for (int64_t s = tid; s < m; s += BD_THREADS) {
          tr_i[base + s] = wc[s] / TC;
          tr_t[base + s] = wc[s] % TC;
        }
      }
      __syncthreads();
      // one warp per cell: every token of the row once, dotted with its query token (a shard: its rows only)
      for (int64_t s = warp; s < (pre ? 0 : m); s += BD_WARPS) {
        const int i = tr_i[base + s];
        const bool own = !P.shard || (i >= own_lo && i < own_hi);
        if (P.mbox && !own) continue;  // (warp-uniform) another rank computes and sends it
        const double v = own ? cell_warp(i, tr_t[base + s]) : 0.0;
        if (lane == 0) {
          if (P.mbox) {
            tr_v[base + s] = v;
            for (int p = 0; p < P.mb_ranks; ++p)
              if (p != my_rank) mbox_publish(peers[p], base + s, v);
          } else if (P.shard) {
            P.xchg[s] = own ? xchg_key(ord_key(v)) : INT64_MIN;
          } else {
            tr_v[base + s] = v;
          }
        }
      }
      if (P.mbox) {
        // the cells of the other ranks' rows arrive in this rank's inbox
        for (int64_t s = tid; s < m; s += BD_THREADS) {
          const int i = tr_i[base + s];
          if (i < own_lo || i >= own_hi) tr_v[base + s] = mbox_wait(peers[my_rank], base + s);
        }
      } else if (P.shard) {
        park(2, CBX_SHARD_WARMUP, base, m);
        return;
      }
      __syncthreads();
      wa_base = base;
      wa_m = m;
    } else {
    // ---------------------------------------------------------- reveal one cell
    i_star = ctrl->i_star;
    t_star = ctrl->t_star;
    const bool own = !P.shard || (i_star >= own_lo && i_star < own_hi);
    const int rc_mode = (RC && rcache) ? ctrl->hit : 2;  // 0 fill the row, 1 served from the cache, 2 on demand
    if (RC && rc_mode != 2) {
      static_assert(CBX_BD_DOC_PREFETCH, "the row fill takes the token range from the decision");
      if constexpr (RC) {
        if (rc_mode == 0) {  // CTA-uniform: all of the row's cells from one gather
          constexpr int KCMAX = (G * VPL) / 4;
          row_cells_mma<T, KCMAX, (KCMAX <= 4 ? 2 : 1)>(
              dtok, ctrl->j0, ctrl->j1, qtok, TC, dim, warp, BD_WARPS, lane, init_cell, P.xmax,
              reinterpret_cast<float*>(bd_smem + P.rc_smem_off), P.rc_cols,
              P.cell_cache + R.trace_off + (int64_t)i_star * TC, t_star, &ctrl->cellkey);
          __syncthreads();
          if (tid == 0) {
            P.row_filled[R.state_off + i_star] = 1;
            ctrl->fills += 1;
          }
        }
      }
    } else if (tokens && own) {
#if CBX_BD_DOC_PREFETCH
      const int64_t j0 = ctrl->j0, j1 = ctrl->j1;
#else
      const int64_t j0 = dto[i_star], j1 = dto[i_star + 1];
#endif
      double best = tokens_max<T, G, VPL, B, WIDE ? CBX_BD_WIDE_BT : 0>(dtok, j0, j1, qtok + (int64_t)t_star * dim, dim,
                                             gid, NGROUPS, sub, init_cell, warp, BD_WARPS, &ctrl->cellkey, &ctrl->lbkey,
                                             P.xmax);
#pragma unroll
      for (int o = 16; o >= G; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, best, o);
        best = w > best ? w : best;
      }
      if (lane == 0) atomicMax(&ctrl->cellkey, (unsigned long long)ord_key(best));
      __syncthreads();
    }
    if (__builtin_expect(P.shard, 0)) {
      if (P.mbox) {
        // the owner sends the cell to every other rank; the others wait for it in their inbox
        if (tid == 0) {
          const int64_t pos = ctrl->n_reveals;
          double v;
          if (own) {
            v = tokens ? ord_val(ctrl->cellkey) : P.matrix[(R.row_begin + i_star) * P.ld_matrix + t_star];
            for (int p = 0; p < P.mb_ranks; ++p)
              if (p != my_rank) mbox_publish(peers[p], pos, v);
          } else {
            v = mbox_wait(peers[my_rank], pos);
          }
          ctrl->cellkey = ord_key(v);
        }
        __syncthreads();
      } else {
        if (tid == 0) {
          const double v = tokens ? ord_val(ctrl->cellkey) : P.matrix[(R.row_begin + i_star) * P.ld_matrix + t_star];
          P.xchg[0] = own ? xchg_key(ord_key(v)) : INT64_MIN;
        }
        park(1, CBX_SHARD_REVEAL, 0, 0);
        return;
      }
    }
    }  // reveal
    } else if (resume_kind == 2) {
      // -------------------------------------------------------- sharded: warm-up values from the exchange
      resume_kind = 0;
      const int64_t base = step->warm_base, m = step->warm_m;
      for (int64_t s = tid; s < m; s += BD_THREADS) tr_v[base + s] = ord_val(xchg_ord(P.xchg[s]));
      __syncthreads();
      wa_base = base;
      wa_m = m;
    } else {
      // -------------------------------------------------------- sharded: the revealed value from the exchange
      resume_kind = 0;
      i_star = ctrl->i_star;
      t_star = ctrl->t_star;
      if (tid == 0) ctrl->cellkey = xchg_ord(P.xchg[0]);
      __syncthreads();
    }
    if (__builtin_expect(wa_m >= 0, 0)) {
      // the one call site of the warm-up's row updates (local cells or cells from the exchange)
      warmup_apply(wa_base, wa_m);
      BD_PHASE(4);
      continue;
    }
    BD_PHASE(2);
    int partner = -1;
    double pre_lo = 0.0, pre_hi = 0.0;
    if (!uniform && warp == 0 && lane < 2) {
      // the exact unrevealed-bound sums of lo (lane 0) and hi (lane 1) at once
      double r;
      if (!exp_add(lane == 0 ? &g_lo[i_star] : &g_hi[i_star], -(lane == 0 ? lo_b : hi_b)[(int64_t)i_star * TC + t_star],
                   &r))
        ctrl->status = 2;
      pre_lo = r;
      pre_hi = __shfl_sync(0x3u, r, 1);
    }
    // the trace entry is written by another warp (tid TRACE_TID): its global stores then never queue in
    // front of thread 0's row update when the SM's load/store unit is busy with another CTA's reveal
    if (tid == (CBX_BD_TRACE_WARP ? 32 : 0)) {
      const double v = (tokens || P.shard) ? ord_val(ctrl->cellkey)
                                           : P.matrix[(R.row_begin + i_star) * P.ld_matrix + t_star];
      const int64_t pos = ctrl->n_reveals;
      tr_i[pos] = i_star;
      tr_t[pos] = t_star;
      tr_v[pos] = v;
      ctrl->n_reveals = pos + 1;
    }
    if (tid == 0) {
      const double v = (tokens || P.shard) ? ord_val(ctrl->cellkey)
                                           : P.matrix[(R.row_begin + i_star) * P.ld_matrix + t_star];
      // what the membership test below reads of OTHER rows, loaded with the row's own state (one round trip)
      const int sw_in = ctrl->swap_in, sw_out = ctrl->swap_out;
      const uint8_t was_member = rv.member[i_star];
      const double p_in = sw_in >= 0 ? rv.proxy[sw_in] : 0.0, p_out = sw_out >= 0 ? rv.proxy[sw_out] : 0.0;
      if (!reveal_update(i_star, t_star, v, !uniform, pre_lo, pre_hi)) ctrl->status = 2;
      // keep the Top-K set equal to the first K of the (-proxy, i) order
      const uint64_t mk = ord_key(last_proxy);
      if (was_member) {
        const int b = sw_in;  // best non-member
        if (b >= 0) {
          const uint64_t bk = ord_key(p_in);
          if (bk > mk || (bk == mk && b < i_star)) {
            rv.member[i_star] = 0;
            rv.member[b] = 1;
            partner = b;
          }
        }
      } else {
        const int w = sw_out;  // worst member
        if (w >= 0) {
          const uint64_t wk = ord_key(p_out);
          if (mk > wk || (mk == wk && i_star < w)) {
            rv.member[i_star] = 1;
            rv.member[w] = 0;
            partner = w;
          }
        }
      }
    }
#ifndef CBX_BD_TREE_PAR
#define CBX_BD_TREE_PAR 1
#endif
#if CBX_BD_TREE_PAR
    if (use_tree) {
      if (tid == 0) ctrl->partner = partner;
      BD_PHASE(6);
      __syncthreads();
      BD_PHASE(7);
      // a member lives in trees 0 (i+) and 3 (worst), a non-member in 1 (i-) and 2 (best non-member);
      // a membership swap touches all four for both rows. Warp s refreshes tree s.
      partner = ctrl->partner;
      const unsigned mask = partner >= 0 ? 0xFu : (rv.member[i_star] ? 0x9u : 0x6u);
      if (warp < 4 && (mask >> warp & 1u)) {
        // i* then the swap partner, through one copy of the walk
        for (int row = i_star, k = 0; k < 2 && row >= 0; ++k, row = partner)
          tree_update_row(tr, rv, N, row, lane, 1u << warp);
      }
    }
#else
    BD_PHASE(6);
    if (use_tree && warp == 0) {
      __syncwarp();
      partner = __shfl_sync(0xffffffffu, partner, 0);
      const unsigned mask = partner >= 0 ? 0xFu : (rv.member[i_star] ? 0x9u : 0x6u);
      tree_update_row(tr, rv, N, i_star, lane, mask);
      if (partner >= 0) tree_update_row(tr, rv, N, partner, lane, 0xFu);
    }
#endif
    __syncthreads();
  }

  // ------------------------------------------------------------ result: Top-K by (-proxy, i)
  if (tid == 0) {
    int32_t* out_k = P.topk + (int64_t)blockIdx.x * P.max_k;
    int cnt = 0;
    for (int i = 0; i < N && cnt < K; ++i) {
      if (!rv.member[i]) continue;
      int p = cnt++;
      const uint64_t mk = ord_key(rv.proxy[i]);
      while (p > 0) {
        const int o = out_k[p - 1];
        const uint64_t ok = ord_key(rv.proxy[o]);
        if (!(mk > ok || (mk == ok && i < o))) break;
        out_k[p] = o;
        --p;
      }
      out_k[p] = i;
    }
    cbx_bandit_out o;
    o.n_reveals = ctrl->n_reveals;
    o.iterations = ctrl->iterations;
    o.terminated_by = term;
    o.status = ctrl->status;
    o.pad = ctrl->fills;  // row-cache variant: rows filled (0 otherwise)
    P.out[blockIdx.x] = o;
    if (P.shard && !P.mbox) {
      step->phase = CBX_SHARD_DONE;
      step->pending = 0;
    }
    if (P.prof) {
      ph[5] = clock64() - tcs;
      for (int k = 0; k < 16; ++k) P.prof[blockIdx.x * 16 + k] = ph[k];
    }
  }
#undef BD_PHASE
}

template <typename T, int G, int VPL>
__global__ void __launch_bounds__(256) warm_cells_kernel(const BanditParams P, int n_runs, const int64_t* wprefix) {
  constexpr int GW = G <= 32 ? G : 32;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = wprefix[n_runs];
  const T* dtok = static_cast<const T*>(P.d_tokens);
  const double init_cell = P.clamp_negative ? 0.0 : -INFINITY;
  for (int64_t g = w0; g < total; g += nw) {
    int lo = 0, hi = n_runs;  // run r with wprefix[r] <= g < wprefix[r + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (wprefix[mid] <= g) lo = mid;
      else hi = mid;
    }
    const cbx_bandit_run_desc& R = P.runs[lo];
    const int64_t slot = R.trace_off + (g - wprefix[lo]);
    const int i = P.trace_i[slot], t = P.trace_t[slot];
    const int64_t* dto = P.d_tok_off + R.row_begin;
    const T* q = static_cast<const T*>(P.q_tokens) + (P.q_tok_off[R.query] + t) * (int64_t)P.dim;
    double best = tokens_max<T, GW, VPL, (VPL == 1 ? 8 : 4), CBX_BD_WARM_BT>(dtok, dto[i], dto[i + 1], q, P.dim, lane / GW,
                                                                   32 / GW, lane % GW, init_cell, 0, 1, nullptr, nullptr,
                                                                   P.xmax);
#pragma unroll
    for (int o = 16; o >= GW; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, best, o);
      best = w > best ? w : best;
    }
    if (lane == 0) P.trace_v[slot] = best;
  }
}

#ifndef CBX_BD_WIDE
#define CBX_BD_WIDE 1  // 512-thread CTAs when the runs fit one per SM
#endif
#ifndef CBX_BD_WREG_MAX_MEAN_ROWS
#define CBX_BD_WREG_MAX_MEAN_ROWS 320  // wide launches: the 256-thread register shape up to this mean document length
#endif
template <typename T, int G, int VPL>
static void (*pick_bandit_rc(bool wide, int sm, bool wreg))(const BanditParams) {
  if constexpr (bd_mma_layout<T, G, VPL>()) {
    if constexpr (G * VPL <= 16) {
      if (wide && wreg)
        return sm == 2 ? bandit_kernel<T, G, VPL, 512, true, 2, true, true>
                       : (sm == 1 ? bandit_kernel<T, G, VPL, 512, true, 1, true, true>
                                  : bandit_kernel<T, G, VPL, 512, true, 0, true, true>);
    }
    if (wide) return sm == 2 ? bandit_kernel<T, G, VPL, 512, true, 2, false, true>
                             : (sm == 1 ? bandit_kernel<T, G, VPL, 512, true, 1, false, true>
                                        : bandit_kernel<T, G, VPL, 512, true, 0, false, true>);
    return sm == 2 ? bandit_kernel<T, G, VPL, 256, true, 2, false, true> : bandit_kernel<T, G, VPL, 256, true, 0, false, true>;
  }
  return nullptr;
}
template <typename T, int G, int VPL, bool UNI>
static void (*pick_bandit(bool wide, int sm, bool wreg))(const BanditParams) {
  if constexpr (bd_mma_layout<T, G, VPL>() && G * VPL <= 16) {
    if (wide && wreg)
      return sm == 2 ? bandit_kernel<T, G, VPL, 512, UNI, 2, true>
                     : (sm == 1 ? bandit_kernel<T, G, VPL, 512, UNI, 1, true> : bandit_kernel<T, G, VPL, 512, UNI, 0, true>);
  }
  if (wide) return sm == 2 ? bandit_kernel<T, G, VPL, 512, UNI, 2>
                           : (sm == 1 ? bandit_kernel<T, G, VPL, 512, UNI, 1> : bandit_kernel<T, G, VPL, 512, UNI, 0>);
  return sm == 2 ? bandit_kernel<T, G, VPL, 256, UNI, 2> : bandit_kernel<T, G, VPL, 256, UNI, 0>;
}

template <typename T, int G, int VPL>
int launch_bandit(const BanditParams& P, int64_t n_runs, size_t smem, cudaStream_t st) {
  // wide: every CTA has an SM to itself — because the runs fit one per SM, or because a run's shared-memory
  // state (pools of ~1600 rows and more) leaves no room for a second CTA anyway (cfg5: 2000 rows)
  const bool wide = CBX_BD_WIDE && (n_runs <= sm_count() || smem > 113 * 1024);
  const int sm = P.use_smem ? 2 : (P.trees_smem ? 1 : 0);  // trees_smem is only set when the runs fit one per SM
  // the register shape stages one tile per warp and step above d = 128 (and spills there): d <= 128 only
  const bool wreg = bd_mma_layout<T, G, VPL>() && G * VPL <= 16 && P.q_tokens != nullptr &&
                    P.mean_doc_rows <= CBX_BD_WREG_MAX_MEAN_ROWS;
  const unsigned threads = wide ? (wreg ? 256 : 512) : 256;
  auto kern = pick_bandit<T, G, VPL, false>(wide, sm, wreg);
  if constexpr (sizeof(T) == 2) {  // the BASELINE configs: 16-bit tokens with generic bounds
    if (P.bounds_lo == nullptr) kern = pick_bandit<T, G, VPL, true>(wide, sm, wreg);
    if (P.bounds_lo == nullptr && P.cell_cache != nullptr && !P.shard) {  // row-cache variant
      auto k2 = pick_bandit_rc<T, G, VPL>(wide, sm, wreg);
      if (k2) kern = k2;
    }
  }
  CBX_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (P.mbox && n_runs > 1) {
    // ranks of one launch wait on each other's mailboxes: they must all be resident at once
    BanditParams Pc = P;
    void* args[] = {&Pc};
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3((unsigned)n_runs),
                                                dim3(threads), args, smem, st);
    if (e != cudaSuccess) return fail(CBX_ECUDA, std::string("bandit_kernel cooperative launch: ") + cudaGetErrorString(e));
    return CBX_OK;
  }
  kern<<<(unsigned)n_runs, threads, smem, st>>>(P);
  CBX_LAUNCH_CHECK("bandit_kernel launch");
  return CBX_OK;
}

// The 16-bit layouts carry the most kernel variants (tensor-core screen, wide shapes, row cache): each group of
// layouts is instantiated in its own translation unit (bandit_<dtype>*.cu) so the build runs them in parallel.
#define CBX_BD_EXTERN_LAUNCH(T)                                                                       \
  extern template int launch_bandit<T, 8, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);    \
  extern template int launch_bandit<T, 16, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);   \
  extern template int launch_bandit<T, 32, 1>(const BanditParams&, int64_t, size_t, cudaStream_t);   \
  extern template int launch_bandit<T, 32, 2>(const BanditParams&, int64_t, size_t, cudaStream_t);   \
  extern template int launch_bandit<T, 32, 4>(const BanditParams&, int64_t, size_t, cudaStream_t);
CBX_BD_EXTERN_LAUNCH(__half)
CBX_BD_EXTERN_LAUNCH(__nv_bfloat16)

// lanes per token row: one 16-byte vector each, up to a warp; longer rows give lanes several vectors
template <typename T>
int dispatch_bandit(const BanditParams& P, int64_t n_runs, size_t smem, cudaStream_t st, int dim) {
  constexpr int PER = 16 / sizeof(T);
  const int nvec = dim / PER;
  if (nvec <= 8) return launch_bandit<T, 8, 1>(P, n_runs, smem, st);
  if (nvec <= 16) return launch_bandit<T, 16, 1>(P, n_runs, smem, st);
  if (nvec <= 32) return launch_bandit<T, 32, 1>(P, n_runs, smem, st);
  if (nvec <= 64) return launch_bandit<T, 32, 2>(P, n_runs, smem, st);
  if (nvec <= 128) return launch_bandit<T, 32, 4>(P, n_runs, smem, st);
  return fail(CBX_EINVAL, "bandit: embedding rows above 2 KiB are not supported");
}


template <typename T>
int dispatch_warm(const BanditParams& P, int n_runs, const int64_t* wprefix, unsigned grid, cudaStream_t st) {
  constexpr int PER = 16 / sizeof(T);
  const int nvec = P.dim / PER;
  auto go = [&](auto kern) -> int {
    kern<<<grid, 256, 0, st>>>(P, n_runs, wprefix);
    CBX_LAUNCH_CHECK("warm_cells_kernel launch");
    return CBX_OK;
  };
  if (nvec <= 8) return go(warm_cells_kernel<T, 8, 1>);
  if (nvec <= 16) return go(warm_cells_kernel<T, 16, 1>);
  if (nvec <= 32) return go(warm_cells_kernel<T, 32, 1>);
  if (nvec <= 64) return go(warm_cells_kernel<T, 32, 2>);
  if (nvec <= 128) return go(warm_cells_kernel<T, 32, 4>);
  return fail(CBX_EINVAL, "bandit: embedding rows above 2 KiB are not supported");
}

// the kernel instantiations are compiled per token dtype (bandit_<dtype>.cu; the 16-bit layouts in three units each)
extern template int dispatch_bandit<float>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
extern template int dispatch_bandit<__half>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
extern template int dispatch_bandit<__nv_bfloat16>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
extern template int dispatch_bandit<double>(const BanditParams&, int64_t, size_t, cudaStream_t, int);
extern template int dispatch_warm<float>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);
extern template int dispatch_warm<__half>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);
extern template int dispatch_warm<__nv_bfloat16>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);
extern template int dispatch_warm<double>(const BanditParams&, int, const int64_t*, unsigned, cudaStream_t);

}  // namespace cbx
