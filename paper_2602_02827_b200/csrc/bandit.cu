// K2 — the Col-Bandit adaptive Top-K loop, one CTA per run, no host round trips.
//
// Replaces colbandit/bandit.py:169-350 (run) together with the ledger and
// reveal (oracle.py:243-329), the interval arithmetic (bounds.py:97-263) and
// numpy's Generator(PCG64) draws. Trace parity with the reference needs:
//   * float64 cells from exact products (fp16/bf16 sums are exact in fp64),
//   * CPython math.fsum semantics for every exactly rounded sum (Expansion),
//   * no FMA contraction and Python's left-to-right evaluation order in the
//     bound arithmetic (this translation unit is built with -fmad=false and
//     spells every operation with an explicit _rn intrinsic),
//   * numpy's PCG64 stream: next32 half-word buffering, Lemire bounded draws
//     with no draw for n == 1, random() = (next64 >> 11) * 2^-53,
//   * the loop's control flow: lazy warm-up counted as an iteration, the
//     exhausted-boundary-row switch, ties to the lower row index.
// Ranking state (proxy / lcb / ucb / Top-K membership) lives in shared memory
// when the pool fits, otherwise in global memory; per-row statistics (count,
// Welford mean / m2, unrevealed-column mask, exact-sum expansions) live in
// global memory and are touched only for the revealed row.
#include "common.cuh"

namespace cbx {

constexpr int BD_THREADS = 256;
constexpr int BD_WARPS = BD_THREADS / 32;
constexpr int BD_CAP = 8;              // exact-sum expansion capacity per row
constexpr int BD_SMEM_ROWS = 4096;     // pools up to this size keep ranking state in smem

struct RowState {
  double mean, m2;
  uint64_t unrev;  // bit t set = column t not yet revealed
  int32_t n, pad;
  Expansion<BD_CAP> obs, lo_un, hi_un;
};

static_assert(sizeof(cbx_bandit_run_desc) == 152, "cbx_bandit_run_desc layout");
static_assert(sizeof(cbx_bandit_out) == 24, "cbx_bandit_out layout");

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
  const cbx_bandit_run_desc* runs;
  const double* bounds_lo;
  const double* bounds_hi;
  const int32_t* warm_cells;
  RowState* rows;
  double* g_rank;      // [total_rows * 3] proxy, lcb, ucb when not in smem
  uint8_t* g_member;   // [total_rows]
  int use_smem;
  int32_t* topk;
  int32_t max_k;
  int32_t* trace_i;
  int32_t* trace_t;
  double* trace_v;
  cbx_bandit_out* out;
};

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

// ----------------------------------------------------------------- keyed reductions
struct KeyIdx {
  double k;
  int32_t i;  // -1 = empty
};

// "a is preferred over b" for the four selections of the loop
enum { SEL_MIN_LCB = 0, SEL_MAX_UCB = 1, SEL_MAX_PROXY = 2, SEL_WORST_PROXY = 3 };

__device__ __forceinline__ bool prefer(int sel, const KeyIdx& a, const KeyIdx& b) {
  if (b.i < 0) return a.i >= 0;
  if (a.i < 0) return false;
  switch (sel) {
    case SEL_MIN_LCB: return a.k < b.k || (a.k == b.k && a.i < b.i);      // argmin (lcb, i)
    case SEL_MAX_UCB: return a.k > b.k || (a.k == b.k && a.i < b.i);      // argmax ucb, lowest i
    case SEL_MAX_PROXY: return a.k > b.k || (a.k == b.k && a.i < b.i);    // first in (-proxy, i)
    default: return a.k < b.k || (a.k == b.k && a.i > b.i);               // last in (-proxy, i)
  }
}

__device__ __forceinline__ KeyIdx shfl_ki(const KeyIdx& v, int off) {
  KeyIdx r;
  r.k = __shfl_xor_sync(0xffffffffu, v.k, off);
  r.i = __shfl_xor_sync(0xffffffffu, v.i, off);
  return r;
}

__device__ __forceinline__ void warp_select(int sel, KeyIdx& v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    KeyIdx w = shfl_ki(v, o);
    if (prefer(sel, w, v)) v = w;
  }
}

// ----------------------------------------------------------------- row arithmetic
// refresh(i) of bandit.py:220-247 / compute_decision_state (bounds.py:244-256)
__device__ void row_interval(const RowState& s, int T, bool uniform, double lo_u, double hi_u, double alpha,
                             double log_term, double& proxy, double& lcb, double& ucb) {
  const int n = s.n;
  const double obs = s.obs.round();
  double lo_sum, hi_sum;
  if (uniform) {
    // fsum of (T - n) copies of a constant == the correctly rounded product
    lo_sum = (T - n) ? __dmul_rn((double)(T - n), lo_u) : 0.0;
    hi_sum = (T - n) ? __dmul_rn((double)(T - n), hi_u) : 0.0;
  } else {
    lo_sum = s.lo_un.round();
    hi_sum = s.hi_un.round();
  }
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
  const double sigma = __dsqrt_rn(__ddiv_rn(pymax(s.m2, 0.0), (double)(n - 1)));
  double rho;
  if (2 * n <= T) rho = __dsub_rn(1.0, __ddiv_rn((double)(n - 1), (double)T));
  else rho = __dmul_rn(__dsub_rn(1.0, __ddiv_rn((double)n, (double)T)), __dadd_rn(1.0, __ddiv_rn(1.0, (double)n)));
  double r = __dmul_rn(alpha, (double)T);
  r = __dmul_rn(r, sigma);
  r = __dmul_rn(r, __dsqrt_rn(__ddiv_rn(__dmul_rn(2.0, log_term), (double)n)));
  r = __dmul_rn(r, __dsqrt_rn(rho));
  lcb = pymin(pymax(h_lo, __dsub_rn(est, r)), h_hi);
  ucb = pymax(pymin(h_hi, __dadd_rn(est, r)), h_lo);
}

// ledger._record (oracle.py:305-314): mask, count, Welford, exact sums
__device__ __forceinline__ bool record(RowState& s, int t, double v, bool uniform, const double* lo_row,
                                       const double* hi_row) {
  s.unrev &= ~(1ull << t);
  s.n += 1;
  const double d = __dsub_rn(v, s.mean);
  s.mean = __dadd_rn(s.mean, __ddiv_rn(d, (double)s.n));
  s.m2 = __dadd_rn(s.m2, __dmul_rn(d, __dsub_rn(v, s.mean)));
  bool ok = s.obs.add(v);
  if (!uniform) {
    ok &= s.lo_un.add(-lo_row[t]);
    ok &= s.hi_un.add(-hi_row[t]);
  }
  return ok;
}

// ----------------------------------------------------------------- cell source
template <typename T>
__device__ __forceinline__ double dot_token(const T* __restrict__ e, const double* __restrict__ q, int dim) {
  double acc = 0.0;
  for (int k = 0; k < dim; ++k) acc = fma(Elem<T>::to_d(e[k]), q[k], acc);
  return acc;
}

// ----------------------------------------------------------------- the kernel
template <typename T>
__global__ void __launch_bounds__(BD_THREADS) bandit_kernel(const BanditParams P) {
  extern __shared__ __align__(16) uint8_t bd_smem[];
  const cbx_bandit_run_desc R = P.runs[blockIdx.x];
  const int N = R.n_rows, TC = R.n_cols, K = R.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool uniform = R.bounds_off < 0;
  const double* lo_b = uniform ? nullptr : P.bounds_lo + R.bounds_off;
  const double* hi_b = uniform ? nullptr : P.bounds_hi + R.bounds_off;
  const bool tokens = P.q_tokens != nullptr;
  const int dim = P.dim;

  // shared layout: control block, reduction scratch, query row, [ranking arrays]
  struct Ctrl {
    int action;       // 0 reveal, 1 stop, 2 warm-up, 3 exhaustion, 4 error
    int i_star, t_star;
    int status;
    int64_t n_reveals;
    int iterations;
    KeyIdx sel[4];
  };
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(bd_smem);
  KeyIdx* red = reinterpret_cast<KeyIdx*>(bd_smem + 128);            // [4][BD_WARPS]
  double* cellred = reinterpret_cast<double*>(red + 4 * BD_WARPS);    // [BD_WARPS]
  double* qrow = cellred + BD_WARPS;                                  // [dim] (token source)
  uint8_t* rank_base = reinterpret_cast<uint8_t*>(qrow + (tokens ? dim : 0));
  double *proxy, *lcb, *ucb;
  uint8_t* member;
  if (P.use_smem) {
    proxy = reinterpret_cast<double*>(rank_base);
    lcb = proxy + N;
    ucb = lcb + N;
    member = reinterpret_cast<uint8_t*>(ucb + N);
  } else {
    proxy = P.g_rank + R.state_off * 3;
    lcb = proxy + N;
    ucb = lcb + N;
    member = P.g_member + R.state_off;
  }
  RowState* rows = P.rows + R.state_off;
  int32_t* tr_i = P.trace_i + R.trace_off;
  int32_t* tr_t = P.trace_t + R.trace_off;
  double* tr_v = P.trace_v + R.trace_off;

  // query / document geometry for the token source
  const T* qtok = nullptr;
  const T* dtok = nullptr;
  const int64_t* dto = nullptr;
  if (tokens) {
    qtok = static_cast<const T*>(P.q_tokens) + P.q_tok_off[R.query] * (int64_t)dim;
    dtok = static_cast<const T*>(P.d_tokens);
    dto = P.d_tok_off + R.row_begin;
  }
  const double init_cell = P.clamp_negative ? 0.0 : -INFINITY;

  // cell value H[i, t]: block-cooperative for the token source
  auto cell_block = [&](int i, int t) -> double {
    if (!tokens) return P.matrix[(R.row_begin + i) * P.ld_matrix + t];
    for (int k = tid; k < dim; k += BD_THREADS) qrow[k] = Elem<T>::to_d(qtok[(int64_t)t * dim + k]);
    __syncthreads();
    const int64_t j0 = dto[i], j1 = dto[i + 1];
    double best = init_cell;
    for (int64_t j = j0 + tid; j < j1; j += BD_THREADS) {
      const double d = dot_token<T>(dtok + j * dim, qrow, dim);
      best = d > best ? d : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, best, o);
      best = w > best ? w : best;
    }
    if (lane == 0) cellred[warp] = best;
    __syncthreads();
    double m = cellred[0];
    for (int w = 1; w < BD_WARPS; ++w) m = cellred[w] > m ? cellred[w] : m;
    __syncthreads();
    return m;
  };

  // cell value computed by one warp (warm-up: many rows in parallel)
  auto cell_warp = [&](int i, int t) -> double {
    if (!tokens) return P.matrix[(R.row_begin + i) * P.ld_matrix + t];
    const T* q = qtok + (int64_t)t * dim;
    const int64_t j0 = dto[i], j1 = dto[i + 1];
    double best = init_cell;
    for (int64_t j = j0 + lane; j < j1; j += 32) {
      const T* e = dtok + j * dim;
      double acc = 0.0;
      for (int k = 0; k < dim; ++k) acc = fma(Elem<T>::to_d(e[k]), Elem<T>::to_d(q[k]), acc);
      best = acc > best ? acc : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, best, o);
      best = w > best ? w : best;
    }
    return best;
  };

  auto refresh = [&](int i, const RowState& s) {
    double px, l, u;
    row_interval(s, TC, uniform, R.lo_uniform, R.hi_uniform, R.alpha_ef, R.log_term, px, l, u);
    proxy[i] = px;
    lcb[i] = l;
    ucb[i] = u;
  };

  // rebuild(): membership = first K rows of the (-proxy, i) order (bandit.py:251-263)
  auto rebuild = [&]() {
    for (int i = tid; i < N; i += BD_THREADS) member[i] = 0;
    __syncthreads();
    for (int r = 0; r < K; ++r) {
      KeyIdx best{0.0, -1};
      for (int i = tid; i < N; i += BD_THREADS) {
        if (member[i]) continue;
        KeyIdx c{proxy[i], i};
        if (prefer(SEL_MAX_PROXY, c, best)) best = c;
      }
      warp_select(SEL_MAX_PROXY, best);
      if (lane == 0) red[warp] = best;
      __syncthreads();
      if (tid == 0) {
        KeyIdx b = red[0];
        for (int w = 1; w < BD_WARPS; ++w)
          if (prefer(SEL_MAX_PROXY, red[w], b)) b = red[w];
        member[b.i] = 1;
      }
      __syncthreads();
    }
  };

  // ------------------------------------------------------------ initial state (all n = 0)
  const uint64_t full_mask = TC >= 64 ? ~0ull : ((1ull << TC) - 1ull);
  for (int i = tid; i < N; i += BD_THREADS) {
    RowState s;
    s.mean = 0.0;
    s.m2 = 0.0;
    s.unrev = full_mask;
    s.n = 0;
    s.pad = 0;
    s.obs.clear();
    s.lo_un.clear();
    s.hi_un.clear();
    if (!uniform) {
      for (int t = 0; t < TC; ++t) {
        s.lo_un.add(lo_b[(int64_t)i * TC + t]);
        s.hi_un.add(hi_b[(int64_t)i * TC + t]);
      }
    }
    rows[i] = s;
    refresh(i, s);
  }
  if (tid == 0) {
    ctrl->status = 0;
    ctrl->n_reveals = 0;
    ctrl->iterations = 0;
  }
  __syncthreads();
  rebuild();

  Pcg64 rng;
  rng.sh = R.rng.state_hi;
  rng.sl = R.rng.state_lo;
  rng.ih = R.rng.inc_hi;
  rng.il = R.rng.inc_lo;
  rng.has32 = R.rng.has_uint32;
  rng.buf = R.rng.uinteger;
  bool warmed = (K == N) || (R.explore_mode == CBX_UNIFORM_ROW);
  const double eps = R.explore_mode == CBX_UNIFORM_ROW ? 1.0 : R.epsilon;
  const int64_t total_cells = (int64_t)N * TC;
  int term = CBX_TERM_SEPARATION;

  while (true) {
    // ---------------------------------------------------------- boundary selection
    KeyIdx acc[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[s] = KeyIdx{0.0, -1};
    for (int i = tid; i < N; i += BD_THREADS) {
      if (member[i]) {
        KeyIdx a{lcb[i], i}, b{proxy[i], i};
        if (prefer(SEL_MIN_LCB, a, acc[0])) acc[0] = a;
        if (prefer(SEL_WORST_PROXY, b, acc[3])) acc[3] = b;
      } else {
        KeyIdx a{ucb[i], i}, b{proxy[i], i};
        if (prefer(SEL_MAX_UCB, a, acc[1])) acc[1] = a;
        if (prefer(SEL_MAX_PROXY, b, acc[2])) acc[2] = b;
      }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      warp_select(s, acc[s]);
      if (lane == 0) red[s * BD_WARPS + warp] = acc[s];
    }
    __syncthreads();
    if (tid == 0) {
      KeyIdx f[4];
      for (int s = 0; s < 4; ++s) {
        f[s] = red[s * BD_WARPS];
        for (int w = 1; w < BD_WARPS; ++w)
          if (prefer(s, red[s * BD_WARPS + w], f[s])) f[s] = red[s * BD_WARPS + w];
        ctrl->sel[s] = f[s];
      }
      ctrl->iterations += 1;
      const int i_plus = f[0].i, i_minus = f[1].i;
      const double ucb_minus = i_minus >= 0 ? f[1].k : -INFINITY;
      int action;
      if (lcb[i_plus] >= ucb_minus) {
        action = 1;
      } else if (!warmed) {
        action = 2;
        warmed = true;
      } else if (ctrl->n_reveals == total_cells) {
        action = 3;
      } else {
        action = 0;
        const double wp = __dsub_rn(ucb[i_plus], lcb[i_plus]);
        const double wm = __dsub_rn(ucb[i_minus], lcb[i_minus]);
        int i_star = wp >= wm ? i_plus : i_minus;
        uint64_t un = rows[i_star].unrev;
        if (!un) {
          i_star = i_star == i_plus ? i_minus : i_plus;
          un = rows[i_star].unrev;
          if (!un) {
            action = 4;
            ctrl->status = 1;
          }
        }
        if (action == 0) {
          int t_star = -1;
          if (rng.random() < eps) {
            uint32_t pos = rng.integers((uint32_t)__popcll(un));
            uint64_t m = un;
            for (uint32_t q = 0; q < pos; ++q) m &= m - 1;  // drop the lowest `pos` set bits
            t_star = __ffsll((long long)m) - 1;
          } else if (uniform) {
            t_star = __ffsll((long long)un) - 1;  // all widths equal: first unrevealed column
          } else {
            // first argmax of the width over the ascending unrevealed columns
            double best = -INFINITY;
            for (int t = 0; t < TC; ++t) {
              if (!((un >> t) & 1ull)) continue;
              const double w = __dsub_rn(hi_b[(int64_t)i_star * TC + t], lo_b[(int64_t)i_star * TC + t]);
              if (w > best) {
                best = w;
                t_star = t;
              }
            }
            if (t_star < 0) t_star = __ffsll((long long)un) - 1;
          }
          ctrl->i_star = i_star;
          ctrl->t_star = t_star;
        }
      }
      ctrl->action = action;
    }
    __syncthreads();
    const int action = ctrl->action;
    if (action == 1) break;
    if (action == 3) {
      term = CBX_TERM_EXHAUSTION;
      break;
    }
    if (action == 4) break;

    if (action == 2) {
      // -------------------------------------------------------- lazy warm-up (bandit.py:285-296)
      warmed = true;
      int64_t base = ctrl->n_reveals;
      int64_t m;
      if (R.explore_mode == CBX_EPSILON_GREEDY) {
        m = N;
        if (tid == 0)
          for (int i = 0; i < N; ++i) {
            tr_i[base + i] = i;
            tr_t[base + i] = (int32_t)rng.integers((uint32_t)TC);
          }
      } else {
        m = R.n_warm;
        const int32_t* wc = P.warm_cells + R.warm_off;
        for (int64_t s = tid; s < m; s += BD_THREADS) {
          tr_i[base + s] = wc[s] / TC;
          tr_t[base + s] = wc[s] % TC;
        }
      }
      __syncthreads();
      for (int64_t s = warp; s < m; s += BD_WARPS) {
        const double v = cell_warp(tr_i[base + s], tr_t[base + s]);
        if (lane == 0) tr_v[base + s] = v;
      }
      __syncthreads();
      if (R.explore_mode == CBX_EPSILON_GREEDY) {
        for (int i = tid; i < N; i += BD_THREADS) {
          RowState s = rows[i];
          if (!record(s, tr_t[base + i], tr_v[base + i], uniform, uniform ? nullptr : lo_b + (int64_t)i * TC,
                      uniform ? nullptr : hi_b + (int64_t)i * TC))
            ctrl->status = 2;
          rows[i] = s;
        }
      } else if (tid == 0) {
        for (int64_t s2 = 0; s2 < m; ++s2) {
          const int i = tr_i[base + s2];
          RowState s = rows[i];
          if (!record(s, tr_t[base + s2], tr_v[base + s2], uniform, uniform ? nullptr : lo_b + (int64_t)i * TC,
                      uniform ? nullptr : hi_b + (int64_t)i * TC))
            ctrl->status = 2;
          rows[i] = s;
        }
      }
      __syncthreads();
      if (m > 0) {
        for (int i = tid; i < N; i += BD_THREADS) refresh(i, rows[i]);
        __syncthreads();
        rebuild();
      }
      if (tid == 0) ctrl->n_reveals = base + m;
      __syncthreads();
      continue;
    }

    // ---------------------------------------------------------- reveal one cell
    const int i_star = ctrl->i_star, t_star = ctrl->t_star;
    const double v0 = cell_block(i_star, t_star);
    if (tid == 0) {
      double v = v0;
      if (!tokens) v = P.matrix[(R.row_begin + i_star) * P.ld_matrix + t_star];
      const int64_t pos = ctrl->n_reveals;
      tr_i[pos] = i_star;
      tr_t[pos] = t_star;
      tr_v[pos] = v;
      ctrl->n_reveals = pos + 1;
      RowState s = rows[i_star];
      if (!record(s, t_star, v, uniform, uniform ? nullptr : lo_b + (int64_t)i_star * TC,
                  uniform ? nullptr : hi_b + (int64_t)i_star * TC))
        ctrl->status = 2;
      rows[i_star] = s;
      refresh(i_star, s);
      // keep the Top-K set equal to the first K of the (-proxy, i) order
      const KeyIdx me{proxy[i_star], i_star};
      if (member[i_star]) {
        const KeyIdx bnm = ctrl->sel[SEL_MAX_PROXY];
        if (bnm.i >= 0 && prefer(SEL_MAX_PROXY, bnm, me)) {
          member[i_star] = 0;
          member[bnm.i] = 1;
        }
      } else {
        const KeyIdx wm = ctrl->sel[SEL_WORST_PROXY];
        if (wm.i >= 0 && prefer(SEL_MAX_PROXY, me, wm)) {
          member[i_star] = 1;
          member[wm.i] = 0;
        }
      }
    }
    __syncthreads();
  }

  // ------------------------------------------------------------ result: Top-K by (-proxy, i)
  if (tid == 0) {
    int32_t* out_k = P.topk + (int64_t)blockIdx.x * P.max_k;
    int cnt = 0;
    for (int i = 0; i < N && cnt < K; ++i) {
      if (!member[i]) continue;
      // insertion sort by (-proxy, i)
      int p = cnt++;
      const KeyIdx me{proxy[i], i};
      while (p > 0) {
        const int o = out_k[p - 1];
        const KeyIdx other{proxy[o], o};
        if (!prefer(SEL_MAX_PROXY, me, other)) break;
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
    o.pad = 0;
    P.out[blockIdx.x] = o;
  }
}

}  // namespace cbx

using namespace cbx;

extern "C" {

size_t cbx_bandit_state_bytes(int64_t total_rows) {
  return align_up(sizeof(RowState) * (size_t)total_rows, 256) + align_up(3 * sizeof(double) * total_rows, 256) +
         align_up((size_t)total_rows, 256);
}

int cbx_bandit_run(const cbx_batch* b, const double* matrix, int64_t ld_matrix, const cbx_bandit_run_desc* runs,
                   int64_t n_runs, int32_t max_rows, const double* bounds_lo, const double* bounds_hi,
                   const int32_t* warm_cells, void* state, size_t state_bytes, int32_t* topk, int32_t max_k,
                   int32_t* trace_i, int32_t* trace_t, double* trace_v, cbx_bandit_out* out, void* stream) {
  if (n_runs <= 0) return CBX_OK;
  if (!runs || !out || !topk || !trace_i || !trace_t || !trace_v || !state)
    return fail(CBX_EINVAL, "bandit: NULL buffer");
  if (!b && !matrix) return fail(CBX_EINVAL, "bandit: need token embeddings or a cell matrix");
  if (n_runs > 0x7FFFFFFF) return fail(CBX_EINVAL, "bandit: too many runs");
  if (max_rows <= 0) return fail(CBX_EINVAL, "bandit: max_rows must be positive");
  BanditParams P;
  P.q_tokens = b ? b->q_tokens : nullptr;
  P.q_tok_off = b ? b->q_tok_off : nullptr;
  P.d_tokens = b ? b->d_tokens : nullptr;
  P.d_tok_off = b ? b->d_tok_off : nullptr;
  P.dim = b ? b->dim : 0;
  P.clamp_negative = b ? b->clamp_negative : 0;
  P.matrix = matrix;
  P.ld_matrix = ld_matrix;
  P.runs = runs;
  P.bounds_lo = bounds_lo;
  P.bounds_hi = bounds_hi;
  P.warm_cells = warm_cells;
  // state layout: RowState[total] | rank[3 * total] | member[total]; the caller sized it with
  // cbx_bandit_state_bytes(total_rows) and gives each run a disjoint state_off range
  const size_t row_sz = sizeof(RowState);
  // recover total_rows from state_bytes (largest t with state_bytes(t) <= state_bytes)
  int64_t lo = 0, hi = (int64_t)(state_bytes / row_sz) + 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (cbx_bandit_state_bytes(mid) <= state_bytes) lo = mid;
    else hi = mid - 1;
  }
  const int64_t total = lo;
  uint8_t* base = static_cast<uint8_t*>(state);
  P.rows = reinterpret_cast<RowState*>(base);
  P.g_rank = reinterpret_cast<double*>(base + align_up(row_sz * (size_t)total, 256));
  P.g_member = base + align_up(row_sz * (size_t)total, 256) + align_up(3 * sizeof(double) * total, 256);
  P.topk = topk;
  P.max_k = max_k;
  P.trace_i = trace_i;
  P.trace_t = trace_t;
  P.trace_v = trace_v;
  P.out = out;
  const int dim = b ? b->dim : 0;
  size_t smem = 128 + sizeof(KeyIdx) * 4 * BD_WARPS + sizeof(double) * BD_WARPS + sizeof(double) * dim;
  smem = align_up(smem, 16);
  P.use_smem = max_rows <= BD_SMEM_ROWS ? 1 : 0;
  if (P.use_smem) smem += (size_t)max_rows * (3 * sizeof(double) + 1);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int dt = b ? b->dtype : CBX_F64;
  auto launch = [&](auto kern) -> int {
    CBX_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)n_runs, BD_THREADS, smem, st>>>(P);
    CBX_LAUNCH_CHECK("bandit_kernel launch");
    return CBX_OK;
  };
  switch (dt) {
    case CBX_F32: return launch(bandit_kernel<float>);
    case CBX_F16: return launch(bandit_kernel<__half>);
    case CBX_BF16: return launch(bandit_kernel<__nv_bfloat16>);
    case CBX_F64: return launch(bandit_kernel<double>);
  }
  return fail(CBX_EINVAL, "bandit: unknown dtype");
}

}  // extern "C"
