/*
 * colbandit_b200.h — C ABI of the B200-native MaxSim / Col-Bandit hot path.
 *
 * The reference (arxiv 2602.02827, package ``colbandit`` 0.1.0) is a pure
 * Python library: it has no FFI of its own. Its hot path sits behind three
 * Python seams, and every entry point below replaces the
 * arithmetic behind one of them:
 *
 *   cbx_maxsim_scores / cbx_topk_* / cbx_rerank_topk
 *       replace Similarity.token_scores + MaxSimOracle.row_values/full_score/
 *       exact_topk (colbandit/oracle.py:57-67, 205-235) for a whole batch of
 *       queries — the exhaustive scorer (P1).
 *   cbx_maxsim_cells_f64
 *       replaces MaxSimOracle.row_values/maxsim (oracle.py:205-220) with
 *       float64-exact cells, plus math.fsum row scores (oracle.py:222-227);
 *       backs baselines.full_rerank (baselines.py:89-97).
 *   cbx_bandit_run
 *       replaces bandit.run (colbandit/bandit.py:169-350) including the
 *       ledger / reveal (oracle.py:243-329), the interval arithmetic
 *       (bounds.py:97-263) and numpy's PCG64 draws — the adaptive loop (P2).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless named host_*; buffers are
 *     caller-owned; nothing is allocated inside a hot call.
 *   - Calls are stream-ordered and asynchronous on ``stream`` (a
 *     cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Return 0 on success. CBX_EINVAL maps to Python ValueError, CBX_ERANGE
 *     to IndexError, everything else to RuntimeError; the message is in
 *     cbx_last_error() (thread-local). No C++ exception crosses the ABI.
 *   - Reentrant per stream; one process per GPU.
 */
#ifndef COLBANDIT_B200_H
#define COLBANDIT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CBX_API __attribute__((visibility("default")))
#else
#define CBX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CBX_ABI_VERSION 1

/* status codes */
#define CBX_OK 0
#define CBX_EINVAL 1    /* invalid argument       -> ValueError   */
#define CBX_ERANGE 2    /* index out of range     -> IndexError   */
#define CBX_ECUDA 3     /* CUDA runtime failure   -> RuntimeError */
#define CBX_EINTERNAL 4 /* device-side status     -> RuntimeError */

/* element types of token buffers */
#define CBX_F32 0
#define CBX_F16 1
#define CBX_BF16 2
#define CBX_F64 3

/* scorer path selection for cbx_maxsim_scores */
#define CBX_PATH_AUTO 0   /* tcgen05 for f16/bf16 with Lq<=128, SIMT otherwise */
#define CBX_PATH_TC 1     /* TMA + tcgen05 + TMEM dense scorer (f16/bf16)       */
#define CBX_PATH_SIMT 2   /* CUDA-core scorer, float64 accumulation (any dtype) */

/* explore modes (colbandit/bandit.py:38 EXPLORE_MODES) */
#define CBX_EPSILON_GREEDY 0
#define CBX_STATIC_WARMUP 1
#define CBX_UNIFORM_ROW 2

/* termination codes */
#define CBX_TERM_SEPARATION 0
#define CBX_TERM_EXHAUSTION 1

/*
 * A batch of queries, each with its own candidate documents, CSR-packed.
 * Query q owns query tokens [q_tok_off[q], q_tok_off[q+1]) of q_tokens and
 * documents [q_doc_off[q], q_doc_off[q+1]); document i owns doc tokens
 * [d_tok_off[i], d_tok_off[i+1]) of d_tokens. Token rows are ``dim``
 * contiguous elements of ``dtype``. Mirrors QueryTokens / DocTokens /
 * MaxSimOracle(query, docs, similarity) (oracle.py:70-144) for many queries.
 * The host-side fields (n_*, max_*) describe the device arrays.
 */
typedef struct cbx_batch {
  const void* q_tokens;
  const int64_t* q_tok_off;   /* [n_queries + 1] */
  const void* d_tokens;
  const int64_t* d_tok_off;   /* [n_docs + 1]    */
  const int64_t* q_doc_off;   /* [n_queries + 1] */
  int64_t n_queries;
  int64_t n_docs;
  int64_t n_q_tokens;
  int64_t n_d_tokens;
  int32_t dim;
  int32_t dtype;              /* CBX_F32 / CBX_F16 / CBX_BF16 / CBX_F64 */
  int32_t clamp_negative;     /* Similarity.clamp_negative (oracle.py:65-66) */
  int32_t max_lq;             /* max query tokens over the batch */
  int64_t max_q_docs;         /* max documents of one query       */
  int64_t max_q_doc_tokens;   /* max candidate tokens of one query */
  float d_norm_max;           /* an upper bound on every document token's L2 norm (cbx_token_norm_max);
                                 required (> 0) by the bandit entry points for f16/bf16 tokens, where it
                                 bounds the fp32 screen of the float64 reveal; ignored elsewhere */
  int32_t reserved;
} cbx_batch;

CBX_API int cbx_abi_version(void);
CBX_API const char* cbx_last_error(void);
/* SM count and compute capability of the current device. */
CBX_API int cbx_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------- P1 */
/* Scratch needed by cbx_maxsim_scores / cbx_topk_* / cbx_rerank_topk. */
CBX_API size_t cbx_workspace_bytes(const cbx_batch* b, int k);

/* Dense MaxSim score of every candidate: scores[i] = sum_t max_j <e_ij, q_t>
 * (float32 accumulate on the tcgen05 path, float64 then rounded on SIMT). */
CBX_API int cbx_maxsim_scores(const cbx_batch* b, float* scores, int path,
                      void* workspace, size_t ws_bytes, void* stream);

/* Per-query Top-K by (-score, local index): ties to the lower index like
 * np.lexsort((arange(N), -S)) (oracle.py:229-235). k must be <= 8192 and
 * <= every query's pool size. topk_idx holds query-local doc indices. */
CBX_API int cbx_topk_f32(const float* scores, const int64_t* q_doc_off, int64_t n_queries,
                 int64_t max_q_docs, int k, int32_t* topk_idx, float* topk_val,
                 void* workspace, size_t ws_bytes, void* stream);
CBX_API int cbx_topk_f64(const double* scores, const int64_t* q_doc_off, int64_t n_queries,
                 int64_t max_q_docs, int k, int32_t* topk_idx, double* topk_val,
                 void* workspace, size_t ws_bytes, void* stream);

/* Scores + Top-K in one stream-ordered call (the exhaustive reranker). */
CBX_API int cbx_rerank_topk(const cbx_batch* b, int k, int path, float* scores,
                    int32_t* topk_idx, float* topk_val,
                    void* workspace, size_t ws_bytes, void* stream);

/* float64-exact cells: cells[i * ld + t] = max_j <e_ij, q_t> (clamped if
 * requested) for every doc i of the batch, t < Lq of its query; optional
 * scores_f64[i] = exactly rounded sum of the row (CPython math.fsum). */
CBX_API int cbx_maxsim_cells_f64(const cbx_batch* b, double* cells, int64_t ld,
                         double* scores_f64, void* stream);

/* Pack candidates of an HBM-resident corpus (ColBanditReranker.fit,
 * reranker.py:86-104) into a contiguous CSR batch: out_doc_off[j + 1] =
 * total tokens of candidates 0..j, out_tokens = their rows in candidate
 * order. cand_ids index the corpus documents; a bad id sets status[0] |= 1
 * (checked by the caller after synchronising). out_capacity is in rows. */
CBX_API int cbx_gather_candidates(const void* corpus_tokens, const int64_t* corpus_doc_off,
                                  int64_t n_corpus_docs, int dim, int dtype,
                                  const int64_t* cand_ids, int64_t n_cand, void* out_tokens,
                                  int64_t out_capacity, int64_t* out_doc_off, int* status,
                                  void* stream);

/* Score candidates of an HBM-resident corpus in place (no candidate copy):
 * the batch's d_tokens / n_d_tokens are the CORPUS token rows, its
 * q_doc_off ranges index cand_ids (corpus document ids, corpus_off = corpus
 * CSR offsets). Documents are streamed by TMA straight from the corpus,
 * packed at 8-row granularity. scores / topk as cbx_rerank_topk; a bad id
 * sets status[0] |= 1. */
CBX_API size_t cbx_corpus_workspace_bytes(int64_t n_queries, int64_t n_cand, int64_t max_q_cands, int k);
CBX_API int cbx_corpus_rerank_topk(const cbx_batch* b, const int64_t* corpus_off, int64_t n_corpus,
                                   const int64_t* cand_ids, int k, float* scores, int32_t* topk_idx,
                                   float* topk_val, int* status, void* workspace, size_t ws_bytes,
                                   void* stream);

/* Static-budget baselines (baselines.py:49-86): sums[i] = exactly rounded
 * (math.fsum) sum of cells[i * ld + cols[i * cells_per_row + j]] over j, the
 * partial sums doc_uniform / doc_top_margin rank rows by (baselines.py:38-41).
 * status[0] |= 1 if an exact-sum expansion overflowed (never for sane data). */
CBX_API int cbx_row_partial_fsum(const double* cells, int64_t ld, const int32_t* cols, int64_t n_rows,
                                 int cells_per_row, double* sums, int* status, void* stream);

/* ---------------------------------------------------------------- Stage 1 */
/* Stage-1 candidate scan, replaces colbandit/pipeline.py:105-158
 * (generate_candidates): for every query-token row r of b->q_tokens (rows of
 * all queries, in order; n_q_tokens rows) and the corpus b->d_tokens
 * (n_d_tokens rows; offsets / q_doc_off are not used), the k_prime corpus
 * tokens of highest float64 similarity (floored at 0 if clamp_negative),
 * ranked by (-similarity, corpus token index) like np.lexsort (pipeline.py:137):
 * nb_tok[r * k_prime + j] = corpus token index, nb_val[...] = similarity.
 * path CBX_PATH_TC (f16/bf16, dim <= 256, k_prime <= 64, >= 8192 corpus
 * tokens) scans once with tcgen05 and refines in float64; it needs
 * corpus_norm_max (cbx_token_norm_max) and, after the stream completes,
 * status[0] != 0 means "re-run with CBX_PATH_SIMT" (list overflow or zero
 * ties under clamping). CBX_PATH_SIMT is float64 on the CUDA cores (any
 * dtype). 1 <= k_prime <= min(8192, n_d_tokens); n_q_tokens <= 65535. */
CBX_API size_t cbx_stage1_workspace_bytes(const cbx_batch* b, int k_prime, int path);
CBX_API int cbx_stage1_topk(const cbx_batch* b, int k_prime, int path, float corpus_norm_max,
                            int64_t* nb_tok, double* nb_val, int* status, void* workspace,
                            size_t ws_bytes, void* stream);
/* *out = max over rows of the L2 norm of a token matrix (rounded up to float). */
CBX_API int cbx_token_norm_max(const void* tokens, int64_t n_tokens, int dim, int dtype, float* out,
                               void* stream);

/* ---------------------------------------------------------------- P2 */
/* numpy PCG64 bit-generator state (np.random.default_rng(seed)
 * .bit_generator.state): 128-bit state and increment plus the buffered
 * 32-bit half. */
typedef struct cbx_pcg64 {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint32_t has_uint32;
  uint32_t uinteger;
} cbx_pcg64;

/* One bandit run (BanditConfig, colbandit/bandit.py:40-76). log_term is
 * RadiusConfig.log_term(N, T) evaluated on the host with math.log
 * (bounds.py:138-143). For CBX_STATIC_WARMUP the host draws the warm-up
 * cells with numpy's Generator.choice (bandit.py:152) and passes them, in
 * draw order, at warm_cells[warm_off ...] together with the generator state
 * after that draw; every other draw happens on the device. */
#define CBX_BANDIT_TREE 1
#define CBX_BANDIT_PREWARMED 2
#define CBX_BANDIT_MAX_COLS 128
#define CBX_BANDIT_EDESC 3
typedef struct cbx_bandit_run_desc {
  int64_t query;          /* token source: query index in the batch           */
  int64_t row_begin;      /* global doc index (token source) or matrix row of row 0 */
  int32_t n_rows;         /* pool size N                                      */
  int32_t n_cols;         /* T (query tokens), 1..128                         */
  int32_t k;              /* Top-K target, 1..N (k == 0 is answered on the host) */
  int32_t explore_mode;   /* CBX_EPSILON_GREEDY / CBX_STATIC_WARMUP / CBX_UNIFORM_ROW */
  int32_t n_warm;         /* static warm-up cell count                        */
  int32_t flags;          /* bit 0 (CBX_BANDIT_TREE): boundary selection through tournament trees
                             (O(log N) per reveal) instead of a full pool scan;
                             bit 1 (CBX_BANDIT_PREWARMED): cbx_bandit_prewarm computed the warm-up
                             cells into trace[trace_off, +m) before the loop kernel runs */
  int64_t warm_off;       /* offset of this run's cells in warm_cells         */
  double alpha_ef;
  double epsilon;
  double log_term;
  int64_t bounds_off;     /* element offset of this run's row-major N x T lo/hi block; -1 = uniform */
  double lo_uniform;      /* generic bounds when bounds_off < 0 (bounds.py:177-180) */
  double hi_uniform;
  int64_t trace_off;      /* offset of this run's N*T trace slots             */
  int64_t state_off;      /* offset (in rows) of this run's per-row state     */
  cbx_pcg64 rng;
} cbx_bandit_run_desc;

typedef struct cbx_bandit_out {
  int64_t n_reveals;
  int32_t iterations;
  int32_t terminated_by;  /* CBX_TERM_* */
  int32_t status;         /* 0 ok; 1 both boundary rows exhausted (RuntimeError in the
                             reference, bandit.py:311-312); 2 exact-sum capacity exceeded;
                             3 (CBX_BANDIT_EDESC) the descriptor breaks the shape contract
                             (n_rows < 1, n_cols outside 1..128, k outside 1..min(n_rows, max_k)):
                             nothing ran (ValueError) */
  int32_t pad;
} cbx_bandit_out;

/* Device scratch for `total_rows` rows over all runs of one call; every run's
 * state_off range must span n_rows + CBX_BANDIT_ROW_SLACK rows. */
#define CBX_BANDIT_ROW_SLACK 64
CBX_API size_t cbx_bandit_state_bytes(int64_t total_rows);

/* Run n_runs independent bandits, one CTA each, entirely on the device.
 * Cell source: token embeddings of ``b`` (cells computed on demand in float64
 * like MaxSimOracle(query, docs), oracle.py:205-215) when b != NULL, else the
 * float64 matrix (MaxSimOracle.from_matrix, oracle.py:146-176) with cell
 * (i, t) of a run at matrix[(row_begin + i) * ld_matrix + t].
 * Outputs: topk[r * max_k + j] ranked by (-proxy, row) (bandit.py:349);
 * trace_{i,t,v}[trace_off + s] in reveal order; out[r]. */
CBX_API int cbx_bandit_run(const cbx_batch* b, const double* matrix, int64_t ld_matrix,
                           const cbx_bandit_run_desc* runs, int64_t n_runs, int32_t max_rows,
                           const double* bounds_lo, const double* bounds_hi,
                           const int32_t* warm_cells, void* state, size_t state_bytes,
                           int32_t* topk, int32_t max_k,
                           int32_t* trace_i, int32_t* trace_t, double* trace_v,
                           cbx_bandit_out* out, void* stream);

/* Warm-up pre-pass for token-backed runs whose flags carry CBX_BANDIT_PREWARMED:
 * draws each run's warm-up cells (epsilon-greedy: one column per row from the
 * run's PCG64 stream; static-warmup: warm_cells) and computes their float64
 * values with a grid of warps (HBM-bound), into trace_{i,t,v}[trace_off + s],
 * s < m. warm_prefix: device int64[n_runs + 1], exclusive prefix sum of each
 * run's pre-warmed cell count (0 for other runs); total_cells = its last entry.
 * Launch it on the same stream before cbx_bandit_run with the same arguments;
 * the loop then replays the draws and uses the values (identical results). */
CBX_API int cbx_bandit_prewarm(const cbx_batch* b, const cbx_bandit_run_desc* runs, int64_t n_runs,
                               const int64_t* warm_prefix, int64_t total_cells, const int32_t* warm_cells,
                               int32_t* trace_i, int32_t* trace_t, double* trace_v, void* stream);

/* Document-sharded Col-Bandit (BASELINE cfg4 over several GPUs).
 * One run whose N documents are split over ranks. Every rank keeps the whole
 * compact run state (row statistics, intervals, selection trees, PCG64 stream)
 * and takes the identical decisions; it holds, and reveals, only the tokens of
 * its own rows [own_lo, own_hi) (``b`` indexes rows globally: documents of
 * other ranks may be empty). A call advances the run to its next exchange
 * point: it applies the cell values of the previous exchange, decides, and
 * writes the cells it owns into ``xchg`` as signed-order keys (INT64_MIN for
 * cells it does not own). Between calls the caller combines ``xchg`` across
 * ranks with an all-reduce MAX, over the slot count named by the int32 at
 * offset 0 of ``step_state`` (CBX_SHARD_REVEAL: 1 slot; CBX_SHARD_WARMUP: the
 * warm-up cells, N for epsilon-greedy or n_warm; CBX_SHARD_DONE: finished,
 * further calls return at once). ``step_state``: CBX_BANDIT_STEP_BYTES of
 * device memory, zeroed before the first call (first = 1). ``xchg``: int64
 * [max(N, n_warm, 1)]. Outputs as cbx_bandit_run once DONE, identical on every
 * rank; the trace is reveal-for-reveal the single-GPU trace. */
#define CBX_BANDIT_STEP_BYTES 256
#define CBX_SHARD_REVEAL 0
#define CBX_SHARD_WARMUP 1
#define CBX_SHARD_DONE 2
CBX_API int cbx_bandit_shard_step(const cbx_batch* b, const double* matrix, int64_t ld_matrix,
                                  const cbx_bandit_run_desc* run, int64_t own_lo, int64_t own_hi, int first,
                                  const double* bounds_lo, const double* bounds_hi, const int32_t* warm_cells,
                                  void* state, size_t state_bytes, void* step_state, int64_t* xchg,
                                  int32_t* topk, int32_t max_k, int32_t* trace_i, int32_t* trace_t,
                                  double* trace_v, cbx_bandit_out* out, void* stream);

/* Document-sharded Col-Bandit in ONE persistent launch per rank (the device-
 * initiated exchange of SURVEY §5 / §7.2(4)): the same replicated-state
 * protocol as cbx_bandit_shard_step, but the owner of a revealed cell stores
 * its value straight into every other rank's inbox (slot = the cell's trace
 * position: value, then a system-scope release store of the slot's flag) and
 * the other ranks spin on an acquire load of their own inbox's flag — no
 * kernel boundary, no host, no collective per iteration. The warm-up cells go
 * the same way (one slot per warm-up cell).
 * An inbox holds N*T slots (cbx_mbox_alloc: one cudaMalloc, so a CUDA IPC
 * handle maps exactly it); its flags must be zero before the launch, and no
 * rank may launch before every rank has zeroed its inbox. ``peers`` (device,
 * [n_local][n_ranks]) gives, for each local rank, every rank's inbox as that
 * rank's CTA addresses it (peer pointers from cbx_ipc_open across processes;
 * plain device pointers when several ranks share one launch, n_local > 1,
 * which is then a cooperative launch so that all of them are resident).
 * runs[c] / own[2c], own[2c+1] (device) describe local rank rank0 + c: the
 * same run (identical descriptor but trace_off/state_off) and its owned rows.
 * Outputs as cbx_bandit_run, identical on every rank: the trace is reveal-for-
 * reveal the single-GPU trace. */
#define CBX_IPC_HANDLE_BYTES 64
typedef struct cbx_mbox_peer {
  double* val;      /* [N*T] cell values by trace position */
  int32_t* flag;    /* [N*T] 1 = value present           */
} cbx_mbox_peer;
CBX_API int cbx_bandit_shard_run(const cbx_batch* b, const double* matrix, int64_t ld_matrix,
                                 const cbx_bandit_run_desc* runs, int32_t n_local, const int64_t* own,
                                 int32_t rank0, int32_t n_ranks, const cbx_mbox_peer* peers, int32_t max_rows,
                                 const double* bounds_lo, const double* bounds_hi, const int32_t* warm_cells,
                                 void* state, size_t state_bytes, int32_t* topk, int32_t max_k,
                                 int32_t* trace_i, int32_t* trace_t, double* trace_v, cbx_bandit_out* out,
                                 void* stream);
/* One inbox of `slots` slots in its own device allocation (*bytes = its size, for the zeroing memset). */
CBX_API int cbx_mbox_alloc(int64_t slots, void** base, size_t* bytes);
CBX_API int cbx_mbox_free(void* base);
/* Zero an inbox's flags (stream-ordered) before a run. */
CBX_API int cbx_mbox_clear(void* base, int64_t slots, void* stream);
/* The (val, flag) view of an inbox allocation (or of a peer's mapping of it). */
CBX_API int cbx_mbox_view(void* base, int64_t slots, cbx_mbox_peer* view);
/* CUDA IPC of an inbox between the ranks' processes (NVLink peer mappings). */
CBX_API int cbx_ipc_get_handle(void* base, void* handle64);
CBX_API int cbx_ipc_open(const void* handle64, void** base);
CBX_API int cbx_ipc_close(void* base);

/* The loop's numpy Generator(PCG64) replica, exposed to pin it against numpy
 * streams (tests/golden/pcg64_streams.json): starting from *state (host
 * struct), draw j is Generator.random() (float64 bits in out[j]) when
 * ops[j] == 0, else Generator.integers(ops[j]) (Lemire with rejection on
 * buffered 32-bit halves; no draw for 1). ops/out/state_out are device
 * pointers; state_out (may be NULL) receives the generator after the draws.
 * Same code as the bandit loop's draws (bandit.py:133-134, 164, 314-315). */
CBX_API int cbx_pcg64_draws(const cbx_pcg64* state, const uint32_t* ops, int64_t n_ops, uint64_t* out,
                            cbx_pcg64* state_out, void* stream);

/* Profiling hook: when set (device pointer to n_runs * 16 uint64), every
 * following cbx_bandit_run writes per-run SM-cycle counters of its phases
 * [scan, decide, reveal, trees, warm-up, total, row update, sync, and the
 * row update's sub-phases setup, Welford, exact sum, interval]; NULL disables. */
CBX_API void cbx_bandit_set_profile(void* counters);

/* Row-cache variant of cbx_bandit_run (optional; reported separately from the on-demand loop):
 * the first adaptive reveal of a row computes ALL of its cells from one gather of the document — what the
 * reference's oracle does on first touch (oracle.py:205-215) — and later reveals of that row read them back.
 * ``cells``: float64 [trace slots of the launch] (same offsets as the trace buffers), ``row_filled``: uint8
 * [state rows of the launch], zeroed by the caller; both device pointers, used by the launches that follow
 * until reset with (NULL, NULL). Token-backed runs with generic bounds only (others run on demand). Traces
 * are identical to the on-demand loop's; cbx_bandit_out.pad returns the number of rows filled. */
CBX_API void cbx_bandit_set_row_cache(double* cells, uint8_t* row_filled);
/* A reveal fills its row when the row already has ``min_revealed`` cells revealed (default 2: the warm-up cell
 * and one adaptive reveal); rows that never get that far are revealed on demand. 0 fills on first touch. */
CBX_API void cbx_bandit_set_row_cache_threshold(int min_revealed);

#ifdef __cplusplus
}
#endif
#endif /* COLBANDIT_B200_H */
