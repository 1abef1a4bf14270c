// K2 — the Col-Bandit loop: host side of the C ABI (launch planning, sharded runs, mailboxes, IPC) and the
// small non-template kernels. The loop kernel itself is in bandit_impl.cuh, instantiated per token dtype in
// bandit_f16*.cu / bandit_bf16*.cu / bandit_f32.cu / bandit_f64.cu.
#include "bandit_impl.cuh"

namespace cbx {

// ----------------------------------------------------------------- warm-up pre-pass
// The lazy warm-up (bandit.py:285-296) is the first reveal of a run: one cell
// per row (epsilon-greedy; columns from the run's own PCG64 stream) or the
// host-drawn static sample. Inside the loop kernel a CTA gathers its N
// documents with 8 warps, one document at a time each — latency bound. Here
// the cells of every pre-warmed run are computed by a grid of warps with many
// documents in flight per SM (HBM bound), straight into the run's trace slots
// [trace_off, trace_off + m); the loop kernel then only replays the draws to
// advance its generator. Same cell function, so the values are the ones the
// loop kernel would compute.
__global__ void warm_draw_kernel(const cbx_bandit_run_desc* __restrict__ runs, int n_runs,
                                 const int32_t* __restrict__ warm_cells, int32_t* tr_i, int32_t* tr_t) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_runs) return;
  const cbx_bandit_run_desc& R = runs[r];
  if (!(R.flags & CBX_BANDIT_PREWARMED)) return;
  int32_t* ti = tr_i + R.trace_off;
  int32_t* tt = tr_t + R.trace_off;
  if (R.explore_mode == CBX_EPSILON_GREEDY) {
    Pcg64 rng;
    rng.sh = R.rng.state_hi;
    rng.sl = R.rng.state_lo;
    rng.ih = R.rng.inc_hi;
    rng.il = R.rng.inc_lo;
    rng.has32 = R.rng.has_uint32;
    rng.buf = R.rng.uinteger;
    for (int i = 0; i < R.n_rows; ++i) {
      ti[i] = i;
      tt[i] = (int32_t)rng.integers((uint32_t)R.n_cols);
    }
  } else {
    const int32_t* wc = warm_cells + R.warm_off;
    for (int s = 0; s < R.n_warm; ++s) {
      ti[s] = wc[s] / R.n_cols;
      tt[s] = wc[s] % R.n_cols;
    }
  }
}

// numpy PCG64 stream check (cbx_pcg64_draws): one thread replays a list of draws with the loop's generator
__global__ void pcg64_draws_kernel(cbx_pcg64 st, const uint32_t* __restrict__ ops, int64_t n_ops, uint64_t* out,
                                   cbx_pcg64* st_out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Pcg64 rng;
  rng.sh = st.state_hi;
  rng.sl = st.state_lo;
  rng.ih = st.inc_hi;
  rng.il = st.inc_lo;
  rng.has32 = st.has_uint32;
  rng.buf = st.uinteger;
  for (int64_t j = 0; j < n_ops; ++j) {
    const uint32_t n = ops[j];
    out[j] = n == 0 ? (uint64_t)__double_as_longlong(rng.random()) : (uint64_t)rng.integers(n);
  }
  if (st_out) {
    cbx_pcg64 o;
    o.state_hi = rng.sh;
    o.state_lo = rng.sl;
    o.inc_hi = rng.ih;
    o.inc_lo = rng.il;
    o.has_uint32 = rng.has32;
    o.uinteger = rng.buf;
    *st_out = o;
  }
}

}  // namespace cbx

using namespace cbx;

static unsigned long long* g_bandit_prof = nullptr;
static double* g_bandit_cell_cache = nullptr;   // row-cache variant (cbx_bandit_set_row_cache)
static uint8_t* g_bandit_row_filled = nullptr;
static int g_bandit_rc_min_count = 2;

static size_t state_parts(int64_t rows, size_t* off_obs, size_t* off_lo, size_t* off_hi, size_t* off_rows) {
  size_t o = 0;
  *off_obs = o;
  o += align_up(sizeof(ExpStore) * (size_t)rows, 256);
  *off_lo = o;
  o += align_up(sizeof(ExpStore) * (size_t)rows, 256);
  *off_hi = o;
  o += align_up(sizeof(ExpStore) * (size_t)rows, 256);
  *off_rows = o;
  o += align_up(ROW_STRIDE * (size_t)rows + 64, 256);
  return o;
}

struct ShardArgs {
  int64_t own_lo, own_hi;
  int first;
  int64_t* xchg;
  void* step;
  // mailbox mode (cbx_bandit_shard_run)
  int mbox, ranks, rank0;
  const cbx_mbox_peer* peers;
  const int64_t* own;
};
static int launch_params(const cbx_batch* b, const double* matrix, int64_t ld_matrix, const cbx_bandit_run_desc* runs,
                         int64_t n_runs, int32_t max_rows, const double* bounds_lo, const double* bounds_hi,
                         const int32_t* warm_cells, void* state, size_t state_bytes, int32_t* topk, int32_t max_k,
                         int32_t* trace_i, int32_t* trace_t, double* trace_v, cbx_bandit_out* out, void* stream,
                         const ShardArgs* sa);

extern "C" {

void cbx_bandit_set_profile(void* counters) { g_bandit_prof = static_cast<unsigned long long*>(counters); }
void cbx_bandit_set_row_cache(double* cells, uint8_t* row_filled) {
  g_bandit_cell_cache = cells;
  g_bandit_row_filled = row_filled;
}
void cbx_bandit_set_row_cache_threshold(int min_revealed) { g_bandit_rc_min_count = min_revealed < 0 ? 0 : min_revealed; }

int cbx_pcg64_draws(const cbx_pcg64* state, const uint32_t* ops, int64_t n_ops, uint64_t* out, cbx_pcg64* state_out,
                    void* stream) {
  if (!state || (n_ops > 0 && (!ops || !out))) return fail(CBX_EINVAL, "pcg64_draws: NULL buffer");
  if (n_ops < 0) return fail(CBX_EINVAL, "pcg64_draws: negative draw count");
  pcg64_draws_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(*state, ops, n_ops, out, state_out);
  CBX_LAUNCH_CHECK("pcg64_draws_kernel launch");
  return CBX_OK;
}

size_t cbx_bandit_state_bytes(int64_t total_rows) {
  size_t a, b, c, d;
  return state_parts(total_rows, &a, &b, &c, &d);
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
  return launch_params(b, matrix, ld_matrix, runs, n_runs, max_rows, bounds_lo, bounds_hi, warm_cells, state,
                       state_bytes, topk, max_k, trace_i, trace_t, trace_v, out, stream, nullptr);
}

int cbx_bandit_shard_step(const cbx_batch* b, const double* matrix, int64_t ld_matrix, const cbx_bandit_run_desc* run,
                          int64_t own_lo, int64_t own_hi, int first, const double* bounds_lo, const double* bounds_hi,
                          const int32_t* warm_cells, void* state, size_t state_bytes, void* step_state,
                          int64_t* xchg, int32_t* topk, int32_t max_k, int32_t* trace_i, int32_t* trace_t,
                          double* trace_v, cbx_bandit_out* out, void* stream) {
  if (!run || !out || !topk || !trace_i || !trace_t || !trace_v || !state || !step_state || !xchg)
    return fail(CBX_EINVAL, "bandit shard: NULL buffer");
  if (!b && !matrix) return fail(CBX_EINVAL, "bandit shard: need token embeddings or a cell matrix");
  if (own_lo < 0 || own_hi < own_lo) return fail(CBX_EINVAL, "bandit shard: bad owned row range");
  ShardArgs sa{own_lo, own_hi, first, xchg, step_state, 0, 0, 0, nullptr, nullptr};
  return launch_params(b, matrix, ld_matrix, run, 1, 0x7FFFFFFF, bounds_lo, bounds_hi, warm_cells, state, state_bytes,
                       topk, max_k, trace_i, trace_t, trace_v, out, stream, &sa);
}

int cbx_bandit_shard_run(const cbx_batch* b, const double* matrix, int64_t ld_matrix, const cbx_bandit_run_desc* runs,
                         int32_t n_local, const int64_t* own, int32_t rank0, int32_t n_ranks,
                         const cbx_mbox_peer* peers, int32_t max_rows, const double* bounds_lo,
                         const double* bounds_hi, const int32_t* warm_cells, void* state, size_t state_bytes,
                         int32_t* topk, int32_t max_k, int32_t* trace_i, int32_t* trace_t, double* trace_v,
                         cbx_bandit_out* out, void* stream) {
  if (!runs || !out || !topk || !trace_i || !trace_t || !trace_v || !state || !own || !peers)
    return fail(CBX_EINVAL, "bandit shard run: NULL buffer");
  if (!b && !matrix) return fail(CBX_EINVAL, "bandit shard run: need token embeddings or a cell matrix");
  if (n_local < 1 || n_ranks < 1 || rank0 < 0 || rank0 + n_local > n_ranks)
    return fail(CBX_EINVAL, "bandit shard run: ranks rank0 .. rank0 + n_local - 1 must lie in [0, n_ranks)");
  if (n_local > sm_count()) return fail(CBX_EINVAL, "bandit shard run: more local ranks than SMs");
  if (max_rows <= 0) return fail(CBX_EINVAL, "bandit shard run: max_rows must be positive");
  ShardArgs sa{0, 0, 1, nullptr, nullptr, 1, n_ranks, rank0, peers, own};
  return launch_params(b, matrix, ld_matrix, runs, n_local, max_rows, bounds_lo, bounds_hi, warm_cells, state,
                       state_bytes, topk, max_k, trace_i, trace_t, trace_v, out, stream, &sa);
}

int cbx_mbox_alloc(int64_t slots, void** base, size_t* bytes) {
  if (slots < 1 || !base || !bytes) return fail(CBX_EINVAL, "mbox_alloc: bad arguments");
  const size_t nb = align_up((size_t)slots * sizeof(double), 256) + align_up((size_t)slots * sizeof(int32_t), 256);
  void* p = nullptr;
  CBX_CUDA_CHECK(cudaMalloc(&p, nb));  // its own allocation, so a CUDA IPC handle maps exactly this inbox
  *base = p;
  *bytes = nb;
  return CBX_OK;
}

int cbx_mbox_clear(void* base, int64_t slots, void* stream) {
  if (!base || slots < 1) return fail(CBX_EINVAL, "mbox_clear: bad arguments");
  uint8_t* flags = static_cast<uint8_t*>(base) + align_up((size_t)slots * sizeof(double), 256);
  CBX_CUDA_CHECK(cudaMemsetAsync(flags, 0, (size_t)slots * sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  return CBX_OK;
}

int cbx_mbox_free(void* base) {
  if (base) CBX_CUDA_CHECK(cudaFree(base));
  return CBX_OK;
}

int cbx_mbox_view(void* base, int64_t slots, cbx_mbox_peer* view) {
  if (!base || slots < 1 || !view) return fail(CBX_EINVAL, "mbox_view: bad arguments");
  view->val = static_cast<double*>(base);
  view->flag = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(base) + align_up((size_t)slots * sizeof(double), 256));
  return CBX_OK;
}

int cbx_ipc_get_handle(void* base, void* handle64) {
  if (!base || !handle64) return fail(CBX_EINVAL, "ipc_get_handle: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == CBX_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  CBX_CUDA_CHECK(cudaIpcGetMemHandle(&h, base));
  std::memcpy(handle64, &h, sizeof(h));
  return CBX_OK;
}

int cbx_ipc_open(const void* handle64, void** base) {
  if (!handle64 || !base) return fail(CBX_EINVAL, "ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  CBX_CUDA_CHECK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return CBX_OK;
}

int cbx_ipc_close(void* base) {
  if (base) CBX_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return CBX_OK;
}

int cbx_bandit_prewarm(const cbx_batch* b, const cbx_bandit_run_desc* runs, int64_t n_runs, const int64_t* warm_prefix,
                       int64_t total_cells, const int32_t* warm_cells, int32_t* trace_i, int32_t* trace_t,
                       double* trace_v, void* stream) {
  if (n_runs <= 0 || total_cells <= 0) return CBX_OK;
  if (!b || !runs || !warm_prefix || !trace_i || !trace_t || !trace_v)
    return fail(CBX_EINVAL, "bandit prewarm: NULL buffer");
  if (n_runs > 0x7FFFFFFF) return fail(CBX_EINVAL, "bandit prewarm: too many runs");
  const size_t es = dtype_size(b->dtype);
  if ((b->dim * es) % 16 != 0) return fail(CBX_EINVAL, "bandit: token rows must be a multiple of 16 bytes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  warm_draw_kernel<<<(unsigned)((n_runs + 127) / 128), 128, 0, st>>>(runs, (int)n_runs, warm_cells, trace_i, trace_t);
  CBX_LAUNCH_CHECK("warm_draw_kernel launch");
  BanditParams P{};
  P.q_tokens = b->q_tokens;
  P.q_tok_off = b->q_tok_off;
  P.d_tokens = b->d_tokens;
  P.d_tok_off = b->d_tok_off;
  P.dim = b->dim;
  P.clamp_negative = b->clamp_negative;
  P.xmax = b->d_norm_max;
  P.mean_doc_rows = b->n_docs > 0 ? (int)std::min<int64_t>(b->n_d_tokens / b->n_docs, 1 << 30) : 0;
  if ((b->dtype == CBX_F16 || b->dtype == CBX_BF16) && !(b->d_norm_max > 0.0f))
    return fail(CBX_EINVAL, "bandit: 16-bit tokens need cbx_batch.d_norm_max > 0 (cbx_token_norm_max)");
  P.runs = runs;
  P.trace_i = trace_i;
  P.trace_t = trace_t;
  P.trace_v = trace_v;
  const int64_t warps = std::min<int64_t>(total_cells, (int64_t)sm_count() * 8 * 4);
  const unsigned grid = (unsigned)((warps + 7) / 8);
  switch (b->dtype) {
    case CBX_F32: return dispatch_warm<float>(P, (int)n_runs, warm_prefix, grid, st);
    case CBX_F16: return dispatch_warm<__half>(P, (int)n_runs, warm_prefix, grid, st);
    case CBX_BF16: return dispatch_warm<__nv_bfloat16>(P, (int)n_runs, warm_prefix, grid, st);
    case CBX_F64: return dispatch_warm<double>(P, (int)n_runs, warm_prefix, grid, st);
  }
  return fail(CBX_EINVAL, "bandit prewarm: unknown dtype");
}

}  // extern "C"

static int launch_params(const cbx_batch* b, const double* matrix, int64_t ld_matrix, const cbx_bandit_run_desc* runs,
                         int64_t n_runs, int32_t max_rows, const double* bounds_lo, const double* bounds_hi,
                         const int32_t* warm_cells, void* state, size_t state_bytes, int32_t* topk, int32_t max_k,
                         int32_t* trace_i, int32_t* trace_t, double* trace_v, cbx_bandit_out* out, void* stream,
                         const ShardArgs* sa) {
  if (b) {
    const size_t es = dtype_size(b->dtype);
    if ((b->dim * es) % 16 != 0) return fail(CBX_EINVAL, "bandit: token rows must be a multiple of 16 bytes");
    if ((b->dtype == CBX_F16 || b->dtype == CBX_BF16) && !(b->d_norm_max > 0.0f))
      return fail(CBX_EINVAL, "bandit: 16-bit tokens need cbx_batch.d_norm_max > 0 (cbx_token_norm_max)");
    if ((reinterpret_cast<uintptr_t>(b->d_tokens) | reinterpret_cast<uintptr_t>(b->q_tokens)) & 15)
      return fail(CBX_EINVAL, "bandit: token buffers must be 16-byte aligned");
  }
  // recover the row capacity the caller sized the state for
  int64_t lo = 0, hi = (int64_t)(state_bytes / 64) + 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (cbx_bandit_state_bytes(mid) <= state_bytes) lo = mid;
    else hi = mid - 1;
  }
  size_t o_obs, o_lo, o_hi, o_rows;
  state_parts(lo, &o_obs, &o_lo, &o_hi, &o_rows);
  uint8_t* base = static_cast<uint8_t*>(state);
  BanditParams P;
  P.q_tokens = b ? b->q_tokens : nullptr;
  P.q_tok_off = b ? b->q_tok_off : nullptr;
  P.d_tokens = b ? b->d_tokens : nullptr;
  P.d_tok_off = b ? b->d_tok_off : nullptr;
  P.dim = b ? b->dim : 0;
  P.clamp_negative = b ? b->clamp_negative : 0;
  P.matrix = matrix;
  P.ld_matrix = ld_matrix;
  P.xmax = b ? b->d_norm_max : 0.0f;
  P.mean_doc_rows = b && b->n_docs > 0 ? (int)std::min<int64_t>(b->n_d_tokens / b->n_docs, 1 << 30) : 0;
  P.runs = runs;
  P.bounds_lo = bounds_lo;
  P.bounds_hi = bounds_hi;
  P.warm_cells = warm_cells;
  P.g_obs = reinterpret_cast<ExpStore*>(base + o_obs);
  P.g_lo = reinterpret_cast<ExpStore*>(base + o_lo);
  P.g_hi = reinterpret_cast<ExpStore*>(base + o_hi);
  P.g_rows = base + o_rows;
  P.topk = topk;
  P.max_k = max_k;
  P.trace_i = trace_i;
  P.trace_t = trace_t;
  P.trace_v = trace_v;
  P.out = out;
  P.prof = g_bandit_prof;
  P.cell_cache = g_bandit_cell_cache;
  P.row_filled = g_bandit_row_filled;
  P.rc_smem_off = 0;
  P.rc_cols = 0;
  P.rc_min_count = g_bandit_rc_min_count;
  P.shard = sa ? 1 : 0;
  P.first = sa ? sa->first : 0;
  P.own_lo = sa ? sa->own_lo : 0;
  P.own_hi = sa ? sa->own_hi : 0;
  P.xchg = sa ? sa->xchg : nullptr;
  P.step = sa ? static_cast<BdStep*>(sa->step) : nullptr;
  P.mbox = sa ? sa->mbox : 0;
  P.mb_ranks = sa ? sa->ranks : 0;
  P.mb_rank0 = sa ? sa->rank0 : 0;
  P.mb_peers = sa ? sa->peers : nullptr;
  P.mb_own = sa ? sa->own : nullptr;
  // widest run of the launch (sizes the per-cell bounds staged in shared memory): the batch's longest query,
  // or the matrix width
  const int64_t max_t = std::min<int64_t>(BD_MAX_T, b ? std::max(b->max_lq, 1) : std::max<int64_t>(ld_matrix, 1));
  size_t smem = 128 + sizeof(Cand) * 4 * 16 + 2 * sizeof(double) * (BD_MAX_T + 1);  // reductions: up to 16 warps
  smem = align_up(smem, 16);
  // a host-stepped sharded run resumes from global state; a mailbox run is one launch like any other
  const bool resumable = sa && !sa->mbox;
  P.use_smem = (max_rows <= BD_SMEM_ROWS && !resumable) ? 1 : 0;
  if (P.use_smem) smem += (size_t)(max_rows + BD_ROW_SLACK) * ROW_STRIDE + 64;
  P.trees_smem = 0;
  if (!P.use_smem && !resumable && CBX_BD_WIDE && n_runs <= sm_count()) {
    // 4 trees x (8-byte key + 4-byte tie) per node; nodes = sum over 32-ary levels
    int64_t nn = 0, sz = ((int64_t)max_rows + 31) / 32;
    for (int l = 0; l < 8; ++l) {
      nn += sz;
      if (sz == 1) break;
      sz = (sz + 31) / 32;
    }
    const size_t tb = align_up((size_t)nn * 4 * 12, 16);
    if (smem + tb <= 220 * 1024) {
      P.trees_smem = 1;
      smem += tb;
    }
  }
  P.bounds_smem = 0;
  P.bounds_smem_off = 0;
  if (!resumable && CBX_BD_WIDE && n_runs <= sm_count() && max_rows <= BD_SMEM_ROWS) {
    // 3 expansions per row, plus lo/hi for up to max_t columns per row when per-cell bounds are given
    const size_t need = (size_t)max_rows * 3 * sizeof(ExpStore) +
                        (bounds_lo ? (size_t)max_rows * max_t * 2 * sizeof(double) : 0);
    const size_t off = align_up(smem, 16);
    if (off + need <= 220 * 1024) {
      P.bounds_smem = 1;
      P.bounds_smem_off = (int64_t)off;
      smem = off + need;
    }
  }

  // the run's document offsets beside its rows, when that keeps the launch's occupancy (two CTAs per SM below
  // 113 KB each, one above)
  P.dto_smem_off = 0;
  if (P.use_smem && b) {
    const size_t off = align_up(smem, 16), need = (size_t)(max_rows + 1) * sizeof(int64_t);
    const size_t cap = smem > 113 * 1024 || n_runs <= sm_count() ? 220 * 1024 : 113 * 1024;
    if (off + need <= cap) {
      P.dto_smem_off = (int64_t)off;
      smem = off + need;
    }
  }

  if (P.cell_cache && b && !sa) {
    // per-warp column front-runners of the row fill: 3 words x 16 warps x columns
    P.rc_cols = (int32_t)((max_t + 7) / 8 * 8);
    const size_t off = align_up(smem, 16), need = (size_t)48 * P.rc_cols * sizeof(float);
    if (off + need > 220 * 1024) return fail(CBX_EINVAL, "bandit row cache: no shared memory left for the column table");
    P.rc_smem_off = (int64_t)off;
    smem = off + need;
  } else {
    P.cell_cache = nullptr;
    P.row_filled = nullptr;
  }

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int dt = b ? b->dtype : CBX_F64;
  const int dim = b ? b->dim : 16;
  switch (dt) {
    case CBX_F32: return dispatch_bandit<float>(P, n_runs, smem, st, dim);
    case CBX_F16: return dispatch_bandit<__half>(P, n_runs, smem, st, dim);
    case CBX_BF16: return dispatch_bandit<__nv_bfloat16>(P, n_runs, smem, st, dim);
    case CBX_F64: return dispatch_bandit<double>(P, n_runs, smem, st, b ? dim : 16);
  }
  return fail(CBX_EINVAL, "bandit: unknown dtype");
}
