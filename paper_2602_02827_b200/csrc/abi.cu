// extern "C" entry points of libcbx.so (declared in include/colbandit_b200.h).
// Argument checking happens here, before any launch; nothing allocates.
#include "common.cuh"

namespace cbx {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return CBX_ECUDA;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

// defined in the kernel translation units
bool tc_supported(const cbx_batch* b);
int launch_maxsim_tc(const cbx_batch* b, float* scores, cudaStream_t stream);
int launch_maxsim_tc_packed(const cbx_batch* b, const int64_t* corpus_off, int64_t n_corpus, const int64_t* cand_ids,
                            float* scores, void* ws, size_t ws_bytes, int* status, cudaStream_t stream);
size_t packed_plan_bytes(int64_t n_cand);
int launch_maxsim_exact(const cbx_batch* b, double* cells, int64_t ld, double* s64, float* s32, cudaStream_t st);
size_t topk_workspace_bytes(int64_t n_queries, int64_t max_q_docs, int K);
int launch_topk_f32(const float* s, const int64_t* off, int64_t nq, int64_t mx, int K, int32_t* ti, float* tv,
                    void* ws, size_t wb, cudaStream_t st);
int launch_topk_f64(const double* s, const int64_t* off, int64_t nq, int64_t mx, int K, int32_t* ti, double* tv,
                    void* ws, size_t wb, cudaStream_t st);

static int check_batch(const cbx_batch* b) {
  if (!b) return fail(CBX_EINVAL, "batch descriptor is NULL");
  if (b->n_queries < 0 || b->n_docs < 0 || b->n_q_tokens < 0 || b->n_d_tokens < 0)
    return fail(CBX_EINVAL, "negative batch sizes");
  if (b->dim <= 0) return fail(CBX_EINVAL, "embedding dim must be positive");
  if (dtype_size(b->dtype) == 0) return fail(CBX_EINVAL, "unknown dtype code " + std::to_string(b->dtype));
  if (b->n_queries > 0 && (!b->q_tokens || !b->q_tok_off || !b->q_doc_off))
    return fail(CBX_EINVAL, "query buffers are NULL");
  if (b->n_docs > 0 && (!b->d_tokens || !b->d_tok_off)) return fail(CBX_EINVAL, "document buffers are NULL");
  if (b->max_lq < 0) return fail(CBX_EINVAL, "max_lq must be non-negative");
  return CBX_OK;
}

}  // namespace cbx

using namespace cbx;

extern "C" {

int cbx_abi_version(void) { return CBX_ABI_VERSION; }

const char* cbx_last_error(void) { return g_last_error.c_str(); }

int cbx_device_info(int* sm, int* major, int* minor) {
  int dev = 0;
  CBX_CUDA_CHECK(cudaGetDevice(&dev));
  if (sm) CBX_CUDA_CHECK(cudaDeviceGetAttribute(sm, cudaDevAttrMultiProcessorCount, dev));
  if (major) CBX_CUDA_CHECK(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev));
  if (minor) CBX_CUDA_CHECK(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev));
  return CBX_OK;
}

size_t cbx_workspace_bytes(const cbx_batch* b, int k) {
  if (!b) return 0;
  return topk_workspace_bytes(b->n_queries, b->max_q_docs, k);
}

int cbx_maxsim_scores(const cbx_batch* b, float* scores, int path, void* ws, size_t ws_bytes, void* stream) {
  (void)ws;
  (void)ws_bytes;
  int rc = check_batch(b);
  if (rc) return rc;
  if (!scores && b->n_docs > 0) return fail(CBX_EINVAL, "scores buffer is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (path == CBX_PATH_AUTO) path = tc_supported(b) ? CBX_PATH_TC : CBX_PATH_SIMT;
  if (path == CBX_PATH_TC) return launch_maxsim_tc(b, scores, st);
  if (path == CBX_PATH_SIMT) return launch_maxsim_exact(b, nullptr, 0, nullptr, scores, st);
  return fail(CBX_EINVAL, "unknown scorer path " + std::to_string(path));
}

int cbx_topk_f32(const float* scores, const int64_t* q_doc_off, int64_t nq, int64_t max_q_docs, int k,
                 int32_t* topk_idx, float* topk_val, void* ws, size_t ws_bytes, void* stream) {
  if (nq > 0 && (!scores || !q_doc_off || (k > 0 && !topk_idx))) return fail(CBX_EINVAL, "Top-K buffers are NULL");
  return launch_topk_f32(scores, q_doc_off, nq, max_q_docs, k, topk_idx, topk_val, ws, ws_bytes,
                         static_cast<cudaStream_t>(stream));
}

int cbx_topk_f64(const double* scores, const int64_t* q_doc_off, int64_t nq, int64_t max_q_docs, int k,
                 int32_t* topk_idx, double* topk_val, void* ws, size_t ws_bytes, void* stream) {
  if (nq > 0 && (!scores || !q_doc_off || (k > 0 && !topk_idx))) return fail(CBX_EINVAL, "Top-K buffers are NULL");
  return launch_topk_f64(scores, q_doc_off, nq, max_q_docs, k, topk_idx, topk_val, ws, ws_bytes,
                         static_cast<cudaStream_t>(stream));
}

int cbx_rerank_topk(const cbx_batch* b, int k, int path, float* scores, int32_t* topk_idx, float* topk_val, void* ws,
                    size_t ws_bytes, void* stream) {
  int rc = cbx_maxsim_scores(b, scores, path, ws, ws_bytes, stream);
  if (rc) return rc;
  return cbx_topk_f32(scores, b->q_doc_off, b->n_queries, b->max_q_docs, k, topk_idx, topk_val, ws, ws_bytes, stream);
}

size_t cbx_corpus_workspace_bytes(int64_t n_queries, int64_t n_cand, int64_t max_q_cands, int k) {
  return align_up(packed_plan_bytes(n_cand), 256) + topk_workspace_bytes(n_queries, max_q_cands, k);
}

int cbx_corpus_rerank_topk(const cbx_batch* b, const int64_t* corpus_off, int64_t n_corpus, const int64_t* cand_ids,
                           int k, float* scores, int32_t* topk_idx, float* topk_val, int* status, void* ws,
                           size_t ws_bytes, void* stream) {
  int rc = check_batch(b);
  if (rc) return rc;
  if (!corpus_off || (b->n_docs && !cand_ids) || !status || !scores) return fail(CBX_EINVAL, "corpus rerank: NULL buffer");
  if (!tc_supported(b))
    return fail(CBX_EINVAL, "corpus rerank needs the tcgen05 path (f16/bf16, Lq <= 128, dim % 8 == 0)");
  if (ws_bytes < cbx_corpus_workspace_bytes(b->n_queries, b->n_docs, b->max_q_docs, k))
    return fail(CBX_EINVAL, "corpus rerank: workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t plan = align_up(packed_plan_bytes(b->n_docs), 256);
  rc = launch_maxsim_tc_packed(b, corpus_off, n_corpus, cand_ids, scores, ws, plan, status, st);
  if (rc) return rc;
  return cbx_topk_f32(scores, b->q_doc_off, b->n_queries, b->max_q_docs, k, topk_idx, topk_val,
                      static_cast<uint8_t*>(ws) + plan, ws_bytes - plan, stream);
}

int cbx_maxsim_cells_f64(const cbx_batch* b, double* cells, int64_t ld, double* scores_f64, void* stream) {
  int rc = check_batch(b);
  if (rc) return rc;
  if (cells && ld < b->max_lq) return fail(CBX_EINVAL, "cell matrix leading dimension smaller than max_lq");
  return launch_maxsim_exact(b, cells, ld, scores_f64, nullptr, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
