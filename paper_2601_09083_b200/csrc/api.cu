// api.cu — host side of the C ABI declared in include/srt.h: validation,
// pool allocation (cudaMallocAsync on the caller's stream), launches, status.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "srt_internal.cuh"

using namespace srt;

// SMs the fused tree step takes beside the scan by default
#ifndef SRT_STEP_OVERLAP_DEFAULT
#define SRT_STEP_OVERLAP_DEFAULT 0
#endif

struct srt_cache {
  srt_config cfg;
  DevCache dev;
  void* pool;           // one allocation holding every array below
  long long* scratch;   // insert work offsets, grown on demand
  int64_t scratch_cap;  // elements
  int2* rowinfo = nullptr;      // verify: per-row (sequence, position)
  unsigned long long* result = nullptr;  // verify: per-row packed winner (pack_cand)
  int64_t row_cap = 0;          // rows the two buffers above can hold
  LmHeadScratch lm{nullptr, nullptr, nullptr, nullptr, 0};  // srt_verify_lmhead: deferred blocks
  int64_t lm_rows = 0;          // rows lm can hold
  void* path = nullptr;         // srt_verify_path: row lists and walk state
  size_t path_cap = 0;
  uint32_t* hubwork = nullptr;  // hub refresh work list [DIRTY_CAP + 1]
  int device;
  uint32_t tag;  // identifies this cache in insert cursors (never 0)
  // the tree step beside the scan (srt_verify_insert_draft_cursor, overlap mode)
  uint32_t* ov = nullptr;       // its state words (tree_step_ov_words)
  size_t ov_cap = 0;
  int32_t ov_sms = -1;          // srt_cache_set_step_overlap (-1: the default)
  // per-kernel timing (srt_profile_enable)
  std::vector<cudaEvent_t> ev;
  std::vector<int32_t> kid;
  int64_t prof_cap = 0, prof_n = 0;
};

namespace {

thread_local char g_err[256] = "no error";

srt_status cuda_fail(cudaError_t e, const char* what) {
  snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return SRT_ERR_CUDA;
}

#define SRT_CUDA(call, what)                         \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// An NVTX range around every public call (visible in nsys / ncu --nvtx
// timelines; a no-op without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SRT_NVTX(name) NvtxRange nvtx_range_(name)

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

srt_status validate(const srt_config* c) {
  if (!c) return SRT_ERR_INVALID_ARG;
  if (c->vocab_size < 2 || c->max_prompts < 1 || c->max_depth < 1) return SRT_ERR_INVALID_CONFIG;
  if (c->max_match_len < 1 || c->max_match_len > c->max_depth || c->max_match_len > 32)
    return SRT_ERR_INVALID_CONFIG;
  if (c->budget_max < 1 || c->budget_max > 64) return SRT_ERR_INVALID_CONFIG;
  if (c->budget_base < 0 || c->budget_base > c->budget_max) return SRT_ERR_INVALID_CONFIG;
  if (c->budget_slope_num < 0 || c->budget_slope_den < 1) return SRT_ERR_INVALID_CONFIG;
  if (!(c->min_path_score >= 0.0)) return SRT_ERR_INVALID_CONFIG;
  if (c->node_capacity < (int64_t)c->max_prompts + 1 || c->node_capacity >= (int64_t)BAD)
    return SRT_ERR_INVALID_CONFIG;
  if (!is_pow2(c->hash_capacity) || c->hash_capacity < 2 * c->node_capacity)
    return SRT_ERR_INVALID_CONFIG;
  // node ids are hash slots and then the P roots: all must stay below BAD
  if (c->hash_capacity + (int64_t)c->max_prompts >= (int64_t)AUX_CHILD0) return SRT_ERR_INVALID_CONFIG;
  if (c->slot_capacity < c->node_capacity || c->slot_capacity >= (int64_t)BAD)
    return SRT_ERR_INVALID_CONFIG;
  if (c->logits_dtype != SRT_BF16 && c->logits_dtype != SRT_F32) return SRT_ERR_INVALID_CONFIG;
  return SRT_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Launch `fn` (returns cudaError_t), bracketed by timing events if profiling.
template <class F>
cudaError_t timed(srt_cache* c, int32_t kernel, cudaStream_t stream, F fn) {
  if (c->prof_n >= c->prof_cap) return fn();
  const int64_t i = c->prof_n++;
  // under stream capture the records become event nodes of the graph
  // (External), re-recorded by every replay -- srt_profile_peek
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  const unsigned fl = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  cudaEventRecordWithFlags(c->ev[2 * i], stream, fl);
  cudaError_t e = fn();
  cudaEventRecordWithFlags(c->ev[2 * i + 1], stream, fl);
  c->kid[i] = kernel;
  return e;
}

}  // namespace

extern "C" {

int srt_abi_version(void) { return SRT_ABI_VERSION; }

const char* srt_error_string(void) { return g_err; }

srt_status srt_cache_create(const srt_config* cfg, void* stream_, srt_cache** out) {
  SRT_NVTX("srt_cache_create");
  if (!out) return SRT_ERR_INVALID_ARG;
  srt_status st = validate(cfg);
  if (st != SRT_OK) return st;
  cudaStream_t stream = (cudaStream_t)stream_;
  const size_t N = cfg->node_capacity, H = cfg->hash_capacity, W = cfg->slot_capacity;
  const size_t NN = H + (size_t)cfg->max_prompts;  // node ids = hash slots, then roots
  size_t off = 0;
  const size_t o_tok = off;     off = align_up(off + NN * 4);
  const size_t o_cnt = off;     off = align_up(off + NN * 4);
  const size_t o_rec = off;     off = align_up(off + NN * 32);
  const size_t o_hash = off;    off = align_up(off + H * sizeof(HashSlot));
  const size_t o_slots = off;   off = align_up(off + W * 4);
  const size_t o_stok = off;    off = align_up(off + W * 4);
  const size_t o_scnt = off;    off = align_up(off + W * 4);
  const size_t o_ctr = off;     off = align_up(off + 2 * 8);
  const size_t o_status = off;  off = align_up(off + 4);
  const size_t o_sched = off;   off = align_up(off + 2 * 4);
  const size_t PP = (size_t)cfg->max_prompts;
  const size_t o_step = off;    off = align_up(off + (6 * PP + 4 + PP * PDIRTY_WORDS) * 4);
  const size_t o_gb = off;      off = align_up(off + (3 * NOISE_BUCKETS + 1) * 4);
  // hub child lists: ~1 slot per 16 nodes' worth of hash, at least 2^12
  size_t HC = 4096;
  while (HC < H / 512 && HC < (1u << 18)) HC <<= 1;
  size_t P2 = 1;  // prompts rounded up to a power of two: equal per-prompt partitions
  while (P2 < (size_t)cfg->max_prompts) P2 <<= 1;
  while (HC < 16 * P2) HC <<= 1;
  const size_t o_hub = off;     off = align_up(off + HC * (4 * 4 + 8 + (size_t)HUB_K * 12));
  const size_t o_dirty = off;   off = align_up(off + (size_t)DIRTY_CAP * 8 + 2 * 4);
  srt_cache* c = new srt_cache();
  c->cfg = *cfg;
  cudaGetDevice(&c->device);
  {
    static std::atomic<uint64_t> serial{0};
    uint64_t z = (uint64_t)(uintptr_t)c ^ (++serial * 0x9E3779B97F4A7C15ull) ^
                 (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    c->tag = (uint32_t)(z ^ (z >> 31)) | 1u;
  }
  cudaError_t e = cudaMallocAsync(&c->pool, off, stream);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMallocAsync(cache pools)");
  }
  char* b = (char*)c->pool;
  DevCache& d = c->dev;
  d.V = cfg->vocab_size; d.P = cfg->max_prompts; d.D = cfg->max_depth; d.L = cfg->max_match_len;
  d.Bmax = cfg->budget_max; d.b0 = cfg->budget_base; d.snum = cfg->budget_slope_num;
  d.sden = cfg->budget_slope_den; d.min_score = cfg->min_path_score;
  d.N = N; d.H = H; d.W = W;
  d.tok = (int32_t*)(b + o_tok);
  d.cnt = (uint32_t*)(b + o_cnt);
  d.rec = (uint4*)(b + o_rec);
  d.hash = (HashSlot*)(b + o_hash);
  d.slots = (uint32_t*)(b + o_slots);
  d.stok = (int32_t*)(b + o_stok);
  d.scnt = (uint32_t*)(b + o_scnt);
  d.ctr = (unsigned long long*)(b + o_ctr);
  d.status = (uint32_t*)(b + o_status);
  d.sched = (uint32_t*)(b + o_sched);
  d.st_pcount = (uint32_t*)(b + o_step);
  d.st_pdone = d.st_pcount + PP;
  d.st_pready = d.st_pdone + PP;
  d.st_pnd = d.st_pready + PP;
  d.st_pnext = d.st_pnd + PP;
  d.st_pfin = d.st_pnext + PP;
  d.st_ndone = d.st_pfin + PP;
  d.pdirty = d.st_ndone + 4;
  d.gbound = (float*)(b + o_gb);
  d.HC = (uint32_t)HC;
  d.hub_shift = 0;
  while (((size_t)1 << (d.hub_shift + 1)) * P2 <= HC) ++d.hub_shift;
  {
    char* hb = b + o_hub;
    d.hub_claim = (unsigned long long*)hb;  hb += HC * 8;
    d.hub_node = (uint32_t*)hb;             hb += HC * 4;
    d.hub_nch = (uint32_t*)hb;              hb += HC * 4;
    d.hub_csum = (uint32_t*)hb;             hb += HC * 4;
    d.hub_len = (uint32_t*)hb;              hb += HC * 4;
    d.hub_child = (uint32_t*)hb;            hb += HC * HUB_K * 4;
    d.hub_tok = (int32_t*)hb;               hb += HC * HUB_K * 4;
    d.hub_cnt = (uint32_t*)hb;
  }
  d.dirty = (uint2*)(b + o_dirty);
  d.dirty_n = (uint32_t*)(d.dirty + DIRTY_CAP);
  c->scratch = nullptr;
  c->scratch_cap = 0;
  if ((e = cudaMemsetAsync(d.sched, 0, 2 * 4, stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(d.st_pcount, 0, (6 * PP + 4 + PP * PDIRTY_WORDS) * 4, stream)) !=
          cudaSuccess ||
      (e = launch_init_cache(d, stream)) != cudaSuccess ||
      (e = launch_noise_bounds(d, stream)) != cudaSuccess) {
    cudaFreeAsync(c->pool, stream);
    delete c;
    return cuda_fail(e, "init kernels");
  }
  *out = c;
  return SRT_OK;
}

srt_status srt_cache_destroy(srt_cache* c, void* stream) {
  SRT_NVTX("srt_cache_destroy");
  if (!c) return SRT_OK;
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  cudaFreeAsync(c->pool, (cudaStream_t)stream);
  if (c->scratch) cudaFreeAsync(c->scratch, (cudaStream_t)stream);
  if (c->rowinfo) cudaFreeAsync(c->rowinfo, (cudaStream_t)stream);
  if (c->result) cudaFreeAsync(c->result, (cudaStream_t)stream);
  if (c->path) cudaFreeAsync(c->path, (cudaStream_t)stream);
  if (c->hubwork) cudaFreeAsync(c->hubwork, (cudaStream_t)stream);
  if (c->lm.cand_x) cudaFreeAsync(c->lm.cand_x, (cudaStream_t)stream);
  if (c->lm.cand_b) cudaFreeAsync(c->lm.cand_b, (cudaStream_t)stream);
  if (c->lm.cand_X) cudaFreeAsync(c->lm.cand_X, (cudaStream_t)stream);
  if (c->lm.cand_n) cudaFreeAsync(c->lm.cand_n, (cudaStream_t)stream);
  if (c->ov) cudaFreeAsync(c->ov, (cudaStream_t)stream);
  delete c;
  return SRT_OK;
}

namespace {
srt_status insert_impl(srt_cache* c, int32_t n, const int32_t* prompt_id, const int32_t* seq_tok,
                       int64_t stride, const int32_t* from, const int32_t* to,
                       const int32_t* floor_, uint32_t* cursor, srt_insert_stats* stats_dev,
                       cudaStream_t stream) {
  if (c->scratch_cap < (int64_t)n + 1) {
    if (c->scratch) SRT_CUDA(cudaFreeAsync(c->scratch, stream), "cudaFreeAsync(scratch)");
    int64_t cap = std::max<int64_t>(4096, 2 * ((int64_t)n + 1));
    SRT_CUDA(cudaMallocAsync(&c->scratch, cap * sizeof(long long), stream), "cudaMallocAsync(scratch)");
    c->scratch_cap = cap;
  }
  if (!c->hubwork)
    SRT_CUDA(cudaMallocAsync(&c->hubwork, ((size_t)DIRTY_CAP * 2 + 1) * 4, stream),
             "cudaMallocAsync(hub work)");
  // cursor path: spans of <= D new positions; longer ones (run-ahead) walk
  const int32_t short_max = cursor ? c->cfg.max_depth : -1;
  SRT_CUDA(timed(c, SRT_K_INSERT_PLAN, stream,
                 [&] {
                   return launch_insert_plan(c->dev, n, prompt_id, from, to, floor_, short_max,
                                             c->scratch, stream);
                 }),
           "insert plan");
  SRT_CUDA(timed(c, SRT_K_INSERT_WALK, stream,
                 [&] {
                   return launch_insert_walk(c->dev, n, prompt_id, seq_tok, stride, from, to,
                                             floor_, stats_dev, c->scratch, stream);
                 }),
           "insert walk");
  if (cursor)
    SRT_CUDA(timed(c, SRT_K_INSERT_CURSOR, stream,
                   [&] {
                     return launch_insert_cursor(c->dev, n, prompt_id, seq_tok, stride, from, to,
                                                 floor_, short_max, cursor, c->tag, stats_dev,
                                                 stream);
                   }),
             "insert cursor");
  SRT_CUDA(timed(c, SRT_K_HUB_REFRESH, stream,
                 [&] {
                   return launch_hub_refresh(c->dev, 0, c->hubwork, c->hubwork + 2 * DIRTY_CAP,
                                             stream);
                 }),
           "hub refresh");
  return SRT_OK;
}
}  // namespace

srt_status srt_insert(srt_cache* c, int32_t n, const int32_t* prompt_id, const int32_t* seq_tok,
                      int64_t stride, const int32_t* from, const int32_t* to,
                      const int32_t* floor_, srt_insert_stats* stats_dev, void* stream_) {
  SRT_NVTX("srt_insert");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!prompt_id || !seq_tok || !from || !to) return SRT_ERR_INVALID_ARG;
  return insert_impl(c, n, prompt_id, seq_tok, stride, from, to, floor_, nullptr, stats_dev,
                     (cudaStream_t)stream_);
}

srt_status srt_insert_cursor(srt_cache* c, int32_t n, const int32_t* prompt_id,
                             const int32_t* seq_tok, int64_t stride, const int32_t* from,
                             const int32_t* to, const int32_t* floor_, uint32_t* cursor,
                             srt_insert_stats* stats_dev, void* stream_) {
  SRT_NVTX("srt_insert_cursor");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!prompt_id || !seq_tok || !from || !to || !cursor) return SRT_ERR_INVALID_ARG;
  if (c->cfg.max_depth > SRT_CURSOR_MAX_DEPTH) return SRT_ERR_INVALID_ARG;
  if (insert_cursor_smem(c->cfg.max_depth) > 200 * 1024) return SRT_ERR_INVALID_ARG;
  return insert_impl(c, n, prompt_id, seq_tok, stride, from, to, floor_, cursor, stats_dev,
                     (cudaStream_t)stream_);
}

srt_status srt_draft(srt_cache* c, int32_t n, const int32_t* prompt_id, const int32_t* seq_tok,
                     int64_t stride, const int32_t* seq_len, const int32_t* pos_base,
                     int32_t* match_len, int32_t* draft_len, int32_t* draft_tok,
                     int32_t* draft_parent, int32_t* draft_depth, int32_t* draft_pos,
                     uint64_t* draft_mask, int64_t* row_offsets, void* stream) {
  SRT_NVTX("srt_draft");
  return srt_draft_cursor(c, n, prompt_id, seq_tok, stride, seq_len, pos_base, nullptr, match_len,
                          draft_len, draft_tok, draft_parent, draft_depth, draft_pos, draft_mask,
                          row_offsets, stream);
}

srt_status srt_draft_cursor(srt_cache* c, int32_t n, const int32_t* prompt_id,
                            const int32_t* seq_tok, int64_t stride, const int32_t* seq_len,
                            const int32_t* pos_base, const uint32_t* cursor, int32_t* match_len,
                            int32_t* draft_len, int32_t* draft_tok, int32_t* draft_parent,
                            int32_t* draft_depth, int32_t* draft_pos, uint64_t* draft_mask,
                            int64_t* row_offsets, void* stream) {
  SRT_NVTX("srt_draft_cursor");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!row_offsets) return SRT_ERR_INVALID_ARG;
  if (n > 0 && (!prompt_id || !seq_tok || !seq_len || !match_len || !draft_len || !draft_tok ||
                !draft_parent || !draft_depth || !draft_pos || !draft_mask))
    return SRT_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0)
    SRT_CUDA(timed(c, SRT_K_DRAFT, st,
                   [&] {
                     return launch_draft(c->dev, n, prompt_id, seq_tok, stride, seq_len, pos_base,
                                         cursor, c->tag, match_len, draft_len, draft_tok,
                                         draft_parent, draft_depth, draft_pos, draft_mask, st);
                   }),
             "draft");
  SRT_CUDA(timed(c, SRT_K_ROW_OFFSETS, st,
                 [&] { return launch_row_offsets(n, draft_len, row_offsets, st); }),
           "row offsets");
  return SRT_OK;
}

namespace {
// The verify scan (rows scratch sized without reading row_offsets back: rows
// <= n * (Bmax + 1)).
srt_status row_buffers(srt_cache* c, const VerifyArgs& a, cudaStream_t stream) {
  const int64_t rows_max = (int64_t)a.n * (c->cfg.budget_max + 1);
  if (c->row_cap < rows_max) {
    if (c->rowinfo) SRT_CUDA(cudaFreeAsync(c->rowinfo, stream), "cudaFreeAsync(rowinfo)");
    if (c->result) SRT_CUDA(cudaFreeAsync(c->result, stream), "cudaFreeAsync(result)");
    const int64_t cap = std::max<int64_t>(rows_max, 4096);
    SRT_CUDA(cudaMallocAsync(&c->rowinfo, cap * sizeof(int2), stream), "cudaMallocAsync(rowinfo)");
    SRT_CUDA(cudaMallocAsync(&c->result, cap * sizeof(unsigned long long), stream),
             "cudaMallocAsync(result)");
    c->row_cap = cap;
  }
  return SRT_OK;
}

srt_status verify_scan(srt_cache* c, const VerifyArgs& a, cudaStream_t stream) {
  const srt_status bs = row_buffers(c, a, stream);
  if (bs != SRT_OK) return bs;
  SRT_CUDA(timed(c, SRT_K_SCAN, stream,
                 [&] { return launch_scan(c->dev, a, false, c->rowinfo, c->result, stream); }),
           "verify scan");
  return SRT_OK;
}

// SMs the fused tree step runs on beside the scan (0: after it, on every SM).
// SRT_STEP_OVERLAP=<SMs> sets it; 0 turns the overlap off.  D <= 32 and the
// rows scan (16-byte aligned rows) only.
int tree_step_overlap_sms(const srt_cache* c, const VerifyArgs& a) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SRT_STEP_OVERLAP");
    env = e ? atoi(e) : -1;
  }
  const int g = c->ov_sms >= 0 ? c->ov_sms : env >= 0 ? env : SRT_STEP_OVERLAP_DEFAULT;
  if (g <= 0 || c->cfg.max_depth > 32 || !scan_cluster_size(c->cfg.vocab_size, a.dtype) ||
      ((uintptr_t)a.logits % 16) != 0 || g >= num_sms())
    return 0;
  return g;
}

srt_status tree_step_overlapped(srt_cache* c, const VerifyArgs& a, int ov_sms,
                                const int32_t* prompt_id, const int32_t* floor_, uint32_t* cursor,
                                srt_insert_stats* stats_dev, const int32_t* pos_base,
                                int32_t* match_len, int32_t* draft_len, int32_t* draft_tok,
                                int32_t* draft_parent, int32_t* draft_depth, int32_t* draft_pos,
                                uint64_t* draft_mask, int64_t* row_offsets, cudaStream_t stream) {
  const srt_status bs = row_buffers(c, a, stream);
  if (bs != SRT_OK) return bs;
  const size_t words = tree_step_ov_words(a.n, c->cfg.max_prompts);
  if (c->ov_cap < words) {
    if (c->ov) SRT_CUDA(cudaFreeAsync(c->ov, stream), "cudaFreeAsync(ov)");
    SRT_CUDA(cudaMallocAsync(&c->ov, words * 4, stream), "cudaMallocAsync(ov)");
    c->ov_cap = words;
  }
  uint32_t* seq_done = tree_step_ov_seq_done(c->ov, a.n, c->cfg.max_prompts);
  // prep -> rowinfo -> scan (all SMs but ov_sms; each CTA triggers its
  // dependents as it starts) -> the step kernel, a programmatic dependent
  // launch: it starts on the free SMs while the scan runs and waits per
  // sequence on the scan's row counters (never on the scan's completion).
  // If the launch is not overlapped it runs after the scan, with the same
  // results: the scan never waits on it.
  SRT_CUDA(launch_step_prep_ov(c->dev, a.n, prompt_id, a.row_offsets, c->ov, stream), "step prep");
  SRT_CUDA(timed(c, SRT_K_SCAN, stream,
                 [&] {
                   cudaError_t e = launch_rowinfo(c->dev, a, c->rowinfo, c->result, stream);
                   if (e != cudaSuccess) return e;
                   return launch_scan_list(c->dev, a, c->rowinfo, nullptr,
                                           tree_step_ov_total(c->ov, a.n, c->cfg.max_prompts),
                                           c->result, stream, seq_done, num_sms() - ov_sms);
                 }),
           "verify scan beside the fused tree step");
  SRT_CUDA(timed(c, SRT_K_TREE_STEP, stream,
                 [&] {
                   return launch_tree_step_ov(c->dev, a, c->result, prompt_id, floor_, cursor,
                                              c->tag, stats_dev, pos_base, match_len, draft_len,
                                              draft_tok, draft_parent, draft_depth, draft_pos,
                                              draft_mask, row_offsets, c->ov, ov_sms, stream);
                 }),
           "fused tree step beside the scan");
  return SRT_OK;
}

// The fused LM-head GEMM + sampler in place of the scan (rows must fit the
// hidden-state buffer: row_offsets[n] <= hidden_rows, unchecked on the host).
srt_status verify_lmhead_scan(srt_cache* c, const VerifyArgs& a, const LmHeadArgs& h,
                              cudaStream_t stream) {
  const srt_status bs = row_buffers(c, a, stream);
  if (bs != SRT_OK) return bs;
  const int64_t rows_max = (int64_t)a.n * (c->cfg.budget_max + 1);
  if (c->lm_rows < rows_max) {
    if (c->lm.cand_x) {
      SRT_CUDA(cudaFreeAsync(c->lm.cand_x, stream), "cudaFreeAsync(lm)");
      SRT_CUDA(cudaFreeAsync(c->lm.cand_b, stream), "cudaFreeAsync(lm)");
      SRT_CUDA(cudaFreeAsync(c->lm.cand_X, stream), "cudaFreeAsync(lm)");
      SRT_CUDA(cudaFreeAsync(c->lm.cand_n, stream), "cudaFreeAsync(lm)");
    }
    const int64_t cap = std::max<int64_t>(rows_max, 4096);
    const size_t esz = c->cfg.logits_dtype == SRT_BF16 ? 2 : 4;
    c->lm.cap = LMHEAD_CAND_CAP;
    SRT_CUDA(cudaMallocAsync(&c->lm.cand_x, (size_t)cap * LMHEAD_CAND_CAP * 64 * esz, stream),
             "cudaMallocAsync(lm candidates)");
    SRT_CUDA(cudaMallocAsync((void**)&c->lm.cand_b, (size_t)cap * LMHEAD_CAND_CAP * 4, stream),
             "cudaMallocAsync(lm candidates)");
    SRT_CUDA(cudaMallocAsync((void**)&c->lm.cand_X, (size_t)cap * LMHEAD_CAND_CAP * 4, stream),
             "cudaMallocAsync(lm candidates)");
    SRT_CUDA(cudaMallocAsync((void**)&c->lm.cand_n, (size_t)cap * 4, stream),
             "cudaMallocAsync(lm candidates)");
    SRT_CUDA(cudaMemsetAsync(c->lm.cand_n, 0, (size_t)cap * 4, stream), "memset(lm)");
    c->lm_rows = cap;
  }
  SRT_CUDA(timed(c, SRT_K_LMHEAD, stream,
                 [&] {
                   cudaError_t e = launch_rowinfo(c->dev, a, c->rowinfo, c->result, stream);
                   if (e != cudaSuccess) return e;
                   return launch_lmhead_sample(c->dev, a, h, c->rowinfo, c->result, c->lm, stream);
                 }),
           "verify lm-head");
  return SRT_OK;
}

srt_status lmhead_args(const srt_cache* c, const void* hidden, int64_t hidden_rows, int32_t K,
                       const void* weight, void* logits_out, LmHeadArgs* h) {
  if (!hidden || !weight || hidden_rows < 1 || K < 8 || K % 8 ||
      (uintptr_t)hidden % 16 || (uintptr_t)weight % 16)
    return SRT_ERR_INVALID_ARG;
  *h = LmHeadArgs{hidden, hidden_rows, K, weight, logits_out};
  return SRT_OK;
}
}  // namespace

srt_status srt_verify_lmhead(srt_cache* c, int32_t n, const void* hidden, int64_t hidden_rows,
                             int32_t hidden_dim, const void* weight, void* logits_out,
                             const int64_t* row_offsets, const int32_t* draft_len,
                             const int32_t* draft_tok, const int32_t* draft_parent,
                             const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed,
                             float temperature, int32_t eos_id, const int32_t* max_new,
                             int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* sampled,
                             int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
                             int32_t* accepted_nodes, uint8_t* finished, void* stream_) {
  SRT_NVTX("srt_verify_lmhead");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth || !seq_id ||
      !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit || !commit_tok ||
      !accepted_nodes || !finished)
    return SRT_ERR_INVALID_ARG;
  LmHeadArgs h;
  srt_status st = lmhead_args(c, hidden, hidden_rows, hidden_dim, weight, logits_out, &h);
  if (st != SRT_OK) return st;
  VerifyArgs a{n,       nullptr,    (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  st = verify_lmhead_scan(c, a, h, stream);
  if (st != SRT_OK) return st;
  SRT_CUDA(timed(c, SRT_K_ACCEPT, stream,
                 [&] { return launch_accept(c->dev, a, c->result, stream); }),
           "verify accept");
  return SRT_OK;
}

srt_status srt_verify_lmhead_insert_cursor(
    srt_cache* c, int32_t n, const void* hidden, int64_t hidden_rows, int32_t hidden_dim,
    const void* weight, void* logits_out, const int64_t* row_offsets, const int32_t* draft_len,
    const int32_t* draft_tok, const int32_t* draft_parent, const int32_t* draft_depth,
    const uint64_t* seq_id, uint64_t seed, float temperature, int32_t eos_id,
    const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* sampled,
    int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok, int32_t* accepted_nodes,
    uint8_t* finished, const int32_t* prompt_id, const int32_t* floor_, uint32_t* cursor,
    srt_insert_stats* stats_dev, void* stream_) {
  SRT_NVTX("srt_verify_lmhead_insert_cursor");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth || !seq_id ||
      !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit || !commit_tok ||
      !accepted_nodes || !finished || !prompt_id || !cursor)
    return SRT_ERR_INVALID_ARG;
  if (c->cfg.max_depth > SRT_CURSOR_MAX_DEPTH) return SRT_ERR_INVALID_ARG;
  if (insert_cursor_smem(c->cfg.max_depth) > 200 * 1024) return SRT_ERR_INVALID_ARG;
  LmHeadArgs h;
  srt_status st = lmhead_args(c, hidden, hidden_rows, hidden_dim, weight, logits_out, &h);
  if (st != SRT_OK) return st;
  VerifyArgs a{n,       nullptr,    (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!c->hubwork)
    SRT_CUDA(cudaMallocAsync(&c->hubwork, ((size_t)DIRTY_CAP * 2 + 1) * 4, stream),
             "cudaMallocAsync(hub work)");
  st = verify_lmhead_scan(c, a, h, stream);
  if (st != SRT_OK) return st;
  SRT_CUDA(timed(c, SRT_K_ACCEPT_INSERT, stream,
                 [&] {
                   return launch_accept_insert(c->dev, a, c->result, prompt_id, floor_, cursor,
                                               c->tag, stats_dev, stream);
                 }),
           "verify accept + insert");
  SRT_CUDA(timed(c, SRT_K_HUB_REFRESH, stream,
                 [&] {
                   return launch_hub_refresh(c->dev, 0, c->hubwork, c->hubwork + 2 * DIRTY_CAP,
                                             stream);
                 }),
           "hub refresh");
  return SRT_OK;
}

srt_status srt_verify(srt_cache* c, int32_t n, const void* logits, const int64_t* row_offsets,
                      const int32_t* draft_len, const int32_t* draft_tok,
                      const int32_t* draft_parent, const int32_t* draft_depth,
                      const uint64_t* seq_id, uint64_t seed, float temperature, int32_t eos_id,
                      const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len,
                      int32_t* sampled, int32_t* accept_len, int32_t* n_commit,
                      int32_t* commit_tok, int32_t* accepted_nodes, uint8_t* finished,
                      void* stream_) {
  SRT_NVTX("srt_verify");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!logits || !row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth ||
      !seq_id || !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit ||
      !commit_tok || !accepted_nodes || !finished)
    return SRT_ERR_INVALID_ARG;
  VerifyArgs a{n,       logits,     (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  const srt_status st = verify_scan(c, a, stream);
  if (st != SRT_OK) return st;
  SRT_CUDA(timed(c, SRT_K_ACCEPT, stream,
                 [&] { return launch_accept(c->dev, a, c->result, stream); }),
           "verify accept");
  return SRT_OK;
}

srt_status srt_verify_insert_cursor(
    srt_cache* c, int32_t n, const void* logits, const int64_t* row_offsets,
    const int32_t* draft_len, const int32_t* draft_tok, const int32_t* draft_parent,
    const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed, float temperature,
    int32_t eos_id, const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len,
    int32_t* sampled, int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
    int32_t* accepted_nodes, uint8_t* finished, const int32_t* prompt_id, const int32_t* floor_,
    uint32_t* cursor, srt_insert_stats* stats_dev, void* stream_) {
  SRT_NVTX("srt_verify_insert_cursor");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!logits || !row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth ||
      !seq_id || !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit ||
      !commit_tok || !accepted_nodes || !finished || !prompt_id || !cursor)
    return SRT_ERR_INVALID_ARG;
  if (c->cfg.max_depth > SRT_CURSOR_MAX_DEPTH) return SRT_ERR_INVALID_ARG;
  if (insert_cursor_smem(c->cfg.max_depth) > 200 * 1024) return SRT_ERR_INVALID_ARG;
  VerifyArgs a{n,       logits,     (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!c->hubwork)
    SRT_CUDA(cudaMallocAsync(&c->hubwork, ((size_t)DIRTY_CAP * 2 + 1) * 4, stream),
             "cudaMallocAsync(hub work)");
  const srt_status st = verify_scan(c, a, stream);
  if (st != SRT_OK) return st;
  SRT_CUDA(timed(c, SRT_K_ACCEPT_INSERT, stream,
                 [&] {
                   return launch_accept_insert(c->dev, a, c->result, prompt_id, floor_, cursor,
                                               c->tag, stats_dev, stream);
                 }),
           "verify accept + insert");
  SRT_CUDA(timed(c, SRT_K_HUB_REFRESH, stream,
                 [&] {
                   return launch_hub_refresh(c->dev, 0, c->hubwork, c->hubwork + 2 * DIRTY_CAP,
                                             stream);
                 }),
           "hub refresh");
  return SRT_OK;
}

srt_status srt_verify_insert_draft_cursor(
    srt_cache* c, int32_t n, const void* logits, const int64_t* row_offsets,
    const int32_t* draft_len, const int32_t* draft_tok, const int32_t* draft_parent,
    const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed, float temperature,
    int32_t eos_id, const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len,
    int32_t* sampled, int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
    int32_t* accepted_nodes, uint8_t* finished, const int32_t* prompt_id, const int32_t* floor_,
    uint32_t* cursor, srt_insert_stats* stats_dev, const int32_t* pos_base, int32_t* next_match_len,
    int32_t* next_draft_len, int32_t* next_draft_tok, int32_t* next_draft_parent,
    int32_t* next_draft_depth, int32_t* next_draft_pos, uint64_t* next_draft_mask,
    int64_t* next_row_offsets, void* stream_) {
  SRT_NVTX("srt_verify_insert_draft_cursor");
  if (!c || n < 0 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!logits || !row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth ||
      !seq_id || !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit ||
      !commit_tok || !accepted_nodes || !finished || !prompt_id || !cursor || !next_match_len ||
      !next_draft_len || !next_draft_tok || !next_draft_parent || !next_draft_depth ||
      !next_draft_pos || !next_draft_mask || !next_row_offsets)
    return SRT_ERR_INVALID_ARG;
  if (c->cfg.max_depth > SRT_CURSOR_MAX_DEPTH) return SRT_ERR_INVALID_ARG;
  if (insert_cursor_smem(c->cfg.max_depth) > 200 * 1024) return SRT_ERR_INVALID_ARG;
  VerifyArgs a{n,       logits,     (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  const int ov_sms = tree_step_overlap_sms(c, a);
  if (ov_sms > 0)
    return tree_step_overlapped(c, a, ov_sms, prompt_id, floor_, cursor, stats_dev, pos_base,
                                next_match_len, next_draft_len, next_draft_tok, next_draft_parent,
                                next_draft_depth, next_draft_pos, next_draft_mask,
                                next_row_offsets, stream);
  const srt_status st = verify_scan(c, a, stream);
  if (st != SRT_OK) return st;
  SRT_CUDA(timed(c, SRT_K_TREE_STEP, stream,
                 [&] {
                   return launch_tree_step(c->dev, a, c->result, prompt_id, floor_, cursor, c->tag,
                                           stats_dev, pos_base, next_match_len, next_draft_len,
                                           next_draft_tok, next_draft_parent, next_draft_depth,
                                           next_draft_pos, next_draft_mask, next_row_offsets,
                                           stream);
                 }),
           "fused tree step");
  return SRT_OK;
}

srt_status srt_cache_set_step_overlap(srt_cache* c, int32_t sms) {
  if (!c || sms < -1 || sms >= num_sms()) return SRT_ERR_INVALID_ARG;
  c->ov_sms = sms;
  return SRT_OK;
}

srt_status srt_verify_path(srt_cache* c, int32_t n, int32_t path_rounds, const void* logits,
                           const int64_t* row_offsets, const int32_t* draft_len,
                           const int32_t* draft_tok, const int32_t* draft_parent,
                           const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed,
                           float temperature, int32_t eos_id, const int32_t* max_new,
                           int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* sampled,
                           int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
                           int32_t* accepted_nodes, uint8_t* finished, void* stream_) {
  SRT_NVTX("srt_verify_path");
  if (!c || n < 0 || stride < 0 || path_rounds < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f) || !(temperature < 3.4e38f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!logits || !row_offsets || !draft_len || !draft_tok || !draft_parent || !draft_depth ||
      !seq_id || !max_new || !seq_tok || !seq_len || !sampled || !accept_len || !n_commit ||
      !commit_tok || !accepted_nodes || !finished)
    return SRT_ERR_INVALID_ARG;
  if (!scan_cluster_size(c->cfg.vocab_size, (int)c->cfg.logits_dtype) ||
      ((uintptr_t)logits % 16) != 0)
    return SRT_ERR_INVALID_ARG;  // (the rows kernel's TMA needs 16-byte rows)
  VerifyArgs a{n,       logits,     (int)c->cfg.logits_dtype, row_offsets, draft_len, draft_tok,
               draft_parent, draft_depth, seq_id, seed,    temperature, eos_id,    max_new,
               seq_tok, stride,     seq_len,  sampled,     accept_len,  n_commit,  commit_tok,
               accepted_nodes, finished};
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t rows_max = (int64_t)n * (c->cfg.budget_max + 1);
  if (c->row_cap < rows_max) {
    if (c->rowinfo) SRT_CUDA(cudaFreeAsync(c->rowinfo, stream), "cudaFreeAsync(rowinfo)");
    if (c->result) SRT_CUDA(cudaFreeAsync(c->result, stream), "cudaFreeAsync(result)");
    const int64_t cap = std::max<int64_t>(rows_max, 4096);
    SRT_CUDA(cudaMallocAsync(&c->rowinfo, cap * sizeof(int2), stream), "cudaMallocAsync(rowinfo)");
    SRT_CUDA(cudaMallocAsync(&c->result, cap * sizeof(unsigned long long), stream),
             "cudaMallocAsync(result)");
    c->row_cap = cap;
  }
  const size_t need = path_scratch_bytes(n, c->cfg.budget_max);
  if (c->path_cap < need) {
    if (c->path) SRT_CUDA(cudaFreeAsync(c->path, stream), "cudaFreeAsync(path)");
    SRT_CUDA(cudaMallocAsync(&c->path, need, stream), "cudaMallocAsync(path)");
    c->path_cap = need;
  }
  SRT_CUDA(timed(c, SRT_K_SCAN, stream,
                 [&] {
                   return launch_path_verify(c->dev, a, c->rowinfo, c->result, c->path,
                                             path_rounds, stream);
                 }),
           "verify path");
  SRT_CUDA(timed(c, SRT_K_ACCEPT, stream,
                 [&] { return launch_accept(c->dev, a, c->result, stream); }),
           "verify accept");
  return SRT_OK;
}

srt_status srt_sample_rows_reference(srt_cache* c, int32_t n, const void* logits,
                                     const int64_t* row_offsets, const int32_t* draft_depth,
                                     const int32_t* seq_len, const uint64_t* seq_id,
                                     uint64_t seed, float temperature, int32_t* sampled,
                                     void* stream) {
  SRT_NVTX("srt_sample_rows_reference");
  if (!c || n < 0) return SRT_ERR_INVALID_ARG;
  if (!(temperature > 0.0f)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!logits || !row_offsets || !draft_depth || !seq_len || !seq_id || !sampled)
    return SRT_ERR_INVALID_ARG;
  VerifyArgs a{};
  a.n = n; a.logits = logits; a.dtype = (int)c->cfg.logits_dtype; a.row_offsets = row_offsets;
  a.draft_depth = draft_depth; a.seq_id = seq_id; a.seed = seed; a.temperature = temperature;
  a.seq_len = seq_len ? const_cast<int32_t*>(seq_len) : nullptr;
  a.sampled = sampled;
  SRT_CUDA(launch_scan(c->dev, a, true, nullptr, nullptr, (cudaStream_t)stream),
           "reference scan");
  return SRT_OK;
}

srt_status srt_cache_status(srt_cache* c, uint32_t* bits, srt_cache_stats* stats, void* stream_) {
  SRT_NVTX("srt_cache_status");
  if (!c) return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  uint32_t h_status = 0;
  unsigned long long h_ctr[2] = {0, 0};
  SRT_CUDA(cudaMemcpyAsync(&h_status, c->dev.status, 4, cudaMemcpyDeviceToHost, stream), "status");
  SRT_CUDA(cudaMemcpyAsync(h_ctr, c->dev.ctr, 16, cudaMemcpyDeviceToHost, stream), "status");
  SRT_CUDA(cudaStreamSynchronize(stream), "status sync");
  if (bits) *bits = h_status;
  if (stats) {
    stats->nodes_used = std::min<unsigned long long>(h_ctr[0], c->dev.N);
    stats->node_capacity = c->dev.N;
    stats->slots_used = std::min<unsigned long long>(h_ctr[1], c->dev.W);
    stats->slot_capacity = c->dev.W;
    stats->hash_capacity = c->dev.H;
  }
  return h_status ? SRT_ERR_DEVICE : SRT_OK;
}

namespace {
// device scratch for the maintenance calls (freed at the end of each call)
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, st); }
};

uint32_t next_tag(uint32_t tag) {
  uint64_t z = (uint64_t)tag * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  return (uint32_t)(z ^ (z >> 31)) | 1u;
}
}  // namespace

srt_status srt_cache_prune(srt_cache* c, int32_t p, uint32_t theta, int64_t* removed_out,
                           void* stream_) {
  SRT_NVTX("srt_cache_prune");
  if (!c || p < -1 || p >= c->cfg.max_prompts) return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  uint32_t bits = 0;
  srt_cache_stats st{};
  srt_status s0 = srt_cache_status(c, &bits, &st, stream);
  if (s0 == SRT_ERR_CUDA) return s0;
  if (bits & SRT_DEV_CAPACITY) return SRT_ERR_DEVICE;
  // frontiers hold at most every live node; [4] counters
  const size_t cap = st.nodes_used + 64;
  DevBuf buf(stream);
  SRT_CUDA(buf.alloc(4 * cap * 4 + 64), "cudaMallocAsync(prune)");
  uint32_t* fk[2] = {(uint32_t*)buf.p, (uint32_t*)buf.p + cap};
  uint32_t* fd[2] = {(uint32_t*)buf.p + 2 * cap, (uint32_t*)buf.p + 3 * cap};
  unsigned* cnt = (unsigned*)((uint32_t*)buf.p + 4 * cap);           // [0] keep, [1] dead
  unsigned long long* removed = (unsigned long long*)(cnt + 4);     // 8-byte aligned
  std::vector<uint32_t> roots;
  for (int32_t q = 0; q < c->cfg.max_prompts; ++q)
    if (p < 0 || q == p) roots.push_back((uint32_t)(c->dev.H + (uint64_t)q));
  SRT_CUDA(cudaMemcpyAsync(fk[0], roots.data(), roots.size() * 4, cudaMemcpyHostToDevice, stream),
           "prune");
  SRT_CUDA(cudaMemsetAsync(removed, 0, 8, stream), "prune");
  int64_t nk = (int64_t)roots.size(), nd = 0;
  int cur = 0;
  while (nk > 0 || nd > 0) {
    SRT_CUDA(cudaMemsetAsync(cnt, 0, 8, stream), "prune");
    SRT_CUDA(launch_prune_level(c->dev, fk[cur], (int32_t)nk, theta, fk[cur ^ 1], cnt,
                                fd[cur ^ 1], cnt + 1, stream), "prune level");
    SRT_CUDA(launch_kill_level(c->dev, fd[cur], (int32_t)nd, fd[cur ^ 1], cnt + 1, removed, stream),
             "kill level");
    unsigned h[2];
    SRT_CUDA(cudaMemcpyAsync(h, cnt, 8, cudaMemcpyDeviceToHost, stream), "prune");
    SRT_CUDA(cudaStreamSynchronize(stream), "prune");
    nk = h[0];
    nd = h[1];
    cur ^= 1;
  }
  unsigned long long h_removed = 0, h_ctr = 0;
  SRT_CUDA(cudaMemcpyAsync(&h_removed, removed, 8, cudaMemcpyDeviceToHost, stream), "prune");
  SRT_CUDA(cudaMemcpyAsync(&h_ctr, c->dev.ctr, 8, cudaMemcpyDeviceToHost, stream), "prune");
  SRT_CUDA(cudaStreamSynchronize(stream), "prune");
  h_ctr -= h_removed;
  SRT_CUDA(cudaMemcpyAsync(c->dev.ctr, &h_ctr, 8, cudaMemcpyHostToDevice, stream), "prune");
  SRT_CUDA(cudaStreamSynchronize(stream), "prune");
  c->tag = next_tag(c->tag);  // cursors may name removed nodes: invalidate all
  SRT_CUDA(cudaMemsetAsync(c->dev.hub_node, 0xFF, (size_t)c->dev.HC * 4, stream), "prune");
  if (removed_out) *removed_out = (int64_t)h_removed;
  return SRT_OK;
}

srt_status srt_cache_evict(srt_cache* c, int64_t max_nodes, int64_t* removed_out,
                           uint32_t* theta_out, void* stream_) {
  SRT_NVTX("srt_cache_evict");
  if (!c || max_nodes < 0) return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  constexpr int NB = 1 << 16;  // exact counts below 65535, one bin above
  DevBuf buf(stream);
  SRT_CUDA(buf.alloc(NB * 8), "cudaMallocAsync(evict)");
  SRT_CUDA(cudaMemsetAsync(buf.p, 0, NB * 8, stream), "evict");
  SRT_CUDA(launch_count_hist(c->dev, (unsigned long long*)buf.p, NB, stream), "count hist");
  std::vector<unsigned long long> hist(NB);
  SRT_CUDA(cudaMemcpyAsync(hist.data(), buf.p, NB * 8, cudaMemcpyDeviceToHost, stream), "evict");
  SRT_CUDA(cudaStreamSynchronize(stream), "evict");
  unsigned long long live = 0;
  for (auto x : hist) live += x;
  if (removed_out) *removed_out = 0;
  if (theta_out) *theta_out = 0;
  if (live <= (unsigned long long)max_nodes) return SRT_OK;
  // smallest theta leaving at most 0.9 * max_nodes nodes (count >= theta)
  const unsigned long long target = (unsigned long long)(0.9 * (double)max_nodes);
  unsigned long long above = 0;
  uint32_t theta = NB - 1;
  for (int b = NB - 1; b >= 1; --b) {
    if (above + hist[b] > target) {
      theta = (uint32_t)b + 1;
      break;
    }
    above += hist[b];
    theta = (uint32_t)b;
  }
  if (theta_out) *theta_out = theta;
  return srt_cache_prune(c, -1, theta, removed_out, stream);
}

srt_status srt_cache_load(srt_cache* c, int32_t p, const srt_dump_record* recs, int64_t n,
                          void* stream_) {
  SRT_NVTX("srt_cache_load");
  if (!c || p < 0 || p >= c->cfg.max_prompts || n < 1 || !recs || recs[0].token != -1)
    return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  // preorder -> levels: (index of the parent in the previous level, token, count)
  struct Lvl { std::vector<int32_t> par, tok; std::vector<unsigned long long> cnt; };
  std::vector<Lvl> lv(1);
  std::vector<std::pair<int32_t, int32_t>> path = {{0, recs[0].n_children}};  // (idx, left)
  for (int64_t k = 1; k < n; ++k) {
    while (!path.empty() && path.back().second == 0) path.pop_back();
    if (path.empty() || recs[k].token < 0 || recs[k].n_children < 0) return SRT_ERR_INVALID_ARG;
    path.back().second -= 1;
    const size_t d = path.size();
    if (lv.size() <= d) lv.resize(d + 1);
    lv[d].par.push_back(path.back().first);
    lv[d].tok.push_back(recs[k].token);
    lv[d].cnt.push_back(recs[k].count);
    path.push_back({(int32_t)lv[d].tok.size() - 1, recs[k].n_children});
  }
  size_t maxn = 1;
  for (auto& l : lv) maxn = std::max(maxn, l.tok.size());
  DevBuf buf(stream);
  SRT_CUDA(buf.alloc(maxn * (4 + 4 + 4 + 8 + 4) + 64), "cudaMallocAsync(load)");
  uint32_t* ids[2] = {(uint32_t*)buf.p, (uint32_t*)buf.p + maxn};
  int32_t* d_par = (int32_t*)((uint32_t*)buf.p + 2 * maxn);
  int32_t* d_tok = d_par + maxn;
  unsigned long long* d_cnt = (unsigned long long*)(((uintptr_t)(d_tok + maxn) + 7) & ~uintptr_t(7));
  const uint32_t root = (uint32_t)(c->dev.H + (uint64_t)p);
  SRT_CUDA(cudaMemcpyAsync(ids[0], &root, 4, cudaMemcpyHostToDevice, stream), "load");
  int cur = 0;
  for (size_t d = 1; d < lv.size(); ++d) {
    const int32_t m = (int32_t)lv[d].tok.size();
    SRT_CUDA(cudaMemcpyAsync(d_par, lv[d].par.data(), m * 4, cudaMemcpyHostToDevice, stream), "load");
    SRT_CUDA(cudaMemcpyAsync(d_tok, lv[d].tok.data(), m * 4, cudaMemcpyHostToDevice, stream), "load");
    SRT_CUDA(cudaMemcpyAsync(d_cnt, lv[d].cnt.data(), m * 8, cudaMemcpyHostToDevice, stream), "load");
    SRT_CUDA(launch_load_level(c->dev, ids[cur], d_par, d_tok, d_cnt, m, ids[cur ^ 1], stream),
             "load level");
    SRT_CUDA(cudaStreamSynchronize(stream), "load");  // the host arrays are reused
    cur ^= 1;
  }
  SRT_CUDA(cudaMemsetAsync(c->dev.hub_node, 0xFF, (size_t)c->dev.HC * 4, stream), "load");
  SRT_CUDA(cudaStreamSynchronize(stream), "load");
  return SRT_OK;
}

srt_status srt_cache_clear_errors(srt_cache* c, void* stream_) {
  if (!c) return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  uint32_t h_status = 0;
  SRT_CUDA(cudaMemcpyAsync(&h_status, c->dev.status, 4, cudaMemcpyDeviceToHost, stream), "status");
  SRT_CUDA(cudaStreamSynchronize(stream), "status sync");
  h_status &= SRT_DEV_CAPACITY;
  SRT_CUDA(cudaMemcpyAsync(c->dev.status, &h_status, 4, cudaMemcpyHostToDevice, stream), "status");
  SRT_CUDA(cudaStreamSynchronize(stream), "status sync");
  return SRT_OK;
}

srt_status srt_profile_enable(srt_cache* c, int64_t capacity) {
  if (!c || capacity < 0) return SRT_ERR_INVALID_ARG;
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  c->ev.assign(2 * capacity, nullptr);
  for (auto& e : c->ev) SRT_CUDA(cudaEventCreate(&e), "cudaEventCreate");
  c->kid.assign(capacity, -1);
  c->prof_cap = capacity;
  c->prof_n = 0;
  return SRT_OK;
}

srt_status srt_profile_read(srt_cache* c, srt_profile_record* host_buf, int64_t cap,
                            int64_t* n_records, void* stream) {
  if (!c || !n_records || cap < 0) return SRT_ERR_INVALID_ARG;
  SRT_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "profile sync");
  const int64_t n = c->prof_n;
  for (int64_t i = 0; i < n && i < cap && host_buf; ++i) {
    float ms = 0.f;
    SRT_CUDA(cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]), "cudaEventElapsedTime");
    host_buf[i] = srt_profile_record{c->kid[i], ms};
  }
  *n_records = n;
  c->prof_n = 0;
  return SRT_OK;
}

srt_status srt_profile_peek(srt_cache* c, srt_profile_record* host_buf, int64_t cap,
                            int64_t* n_records, void* stream) {
  if (!c || !n_records || cap < 0) return SRT_ERR_INVALID_ARG;
  SRT_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "profile sync");
  const int64_t n = c->prof_n;
  for (int64_t i = 0; i < n && i < cap && host_buf; ++i) {
    float ms = 0.f;
    SRT_CUDA(cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]), "cudaEventElapsedTime");
    host_buf[i] = srt_profile_record{c->kid[i], ms};
  }
  *n_records = n;
  return SRT_OK;
}

srt_status srt_debug_draft_profile(int64_t* dev_buf) {
  SRT_CUDA(set_draft_profile((long long*)dev_buf), "set_draft_profile");
  return SRT_OK;
}

srt_status srt_debug_insert_profile(int64_t* dev_buf) {
  SRT_CUDA(set_insert_profile((long long*)dev_buf), "set_insert_profile");
  return SRT_OK;
}

// ---- multi-GPU exchange records (exchange.cu)
srt_status srt_pack_drafts(int32_t n, int32_t Bmax, const int32_t* match_len,
                           const int32_t* draft_len, const int32_t* draft_tok,
                           const int32_t* draft_parent, const int32_t* draft_depth,
                           const uint64_t* draft_mask, int32_t* records, void* stream) {
  SRT_NVTX("srt_pack_drafts");
  if (n < 0 || Bmax < 1 || Bmax > 64) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!match_len || !draft_len || !draft_tok || !draft_parent || !draft_depth || !draft_mask ||
      !records)
    return SRT_ERR_INVALID_ARG;
  SRT_CUDA(launch_pack_drafts(n, Bmax, match_len, draft_len, draft_tok, draft_parent, draft_depth,
                              draft_mask, records, (cudaStream_t)stream),
           "pack drafts");
  return SRT_OK;
}

srt_status srt_unpack_drafts(int32_t n, int32_t Bmax, const int32_t* records, const int32_t* src,
                             const int32_t* pos_base, int32_t* match_len, int32_t* draft_len,
                             int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                             int32_t* draft_pos, uint64_t* draft_mask, int64_t* row_offsets,
                             void* stream) {
  SRT_NVTX("srt_unpack_drafts");
  if (n < 0 || Bmax < 1 || Bmax > 64 || !row_offsets) return SRT_ERR_INVALID_ARG;
  if (n > 0 && (!records || !src || !match_len || !draft_len || !draft_tok || !draft_parent ||
                !draft_depth || !draft_pos || !draft_mask))
    return SRT_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0)
    SRT_CUDA(launch_unpack_drafts(n, Bmax, records, src, pos_base, match_len, draft_len, draft_tok,
                                  draft_parent, draft_depth, draft_pos, draft_mask, st),
             "unpack drafts");
  SRT_CUDA(launch_row_offsets(n, draft_len, row_offsets, st), "row offsets");
  return SRT_OK;
}

srt_status srt_pack_spans(int32_t n, int32_t Bmax, const int32_t* n_commit,
                          const int32_t* commit_tok, int32_t* records, void* stream) {
  SRT_NVTX("srt_pack_spans");
  if (n < 0 || Bmax < 1 || Bmax > 64) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!n_commit || !commit_tok || !records) return SRT_ERR_INVALID_ARG;
  SRT_CUDA(launch_pack_spans(n, Bmax, n_commit, commit_tok, records, (cudaStream_t)stream),
           "pack spans");
  return SRT_OK;
}

srt_status srt_apply_spans(int32_t n, int32_t Bmax, const int32_t* records, const int32_t* src,
                           int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* from,
                           int32_t* to, void* stream) {
  SRT_NVTX("srt_apply_spans");
  if (n < 0 || Bmax < 1 || Bmax > 64 || stride < 0) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  if (!records || !src || !seq_tok || !seq_len || !from || !to) return SRT_ERR_INVALID_ARG;
  SRT_CUDA(launch_apply_spans(n, Bmax, records, src, seq_tok, stride, seq_len, from, to,
                              (cudaStream_t)stream),
           "apply spans");
  return SRT_OK;
}

srt_status srt_noise_table(float* out, void* stream) {
  if (!out) return SRT_ERR_INVALID_ARG;
  SRT_CUDA(launch_noise_table(out, (cudaStream_t)stream), "noise table");
  return SRT_OK;
}

srt_status srt_log_det_range(uint32_t first_bits, int64_t n, float* out, void* stream) {
  if (!out || n < 0 || (uint64_t)first_bits + (uint64_t)n > (1ull << 32)) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  SRT_CUDA(launch_log_det_range(first_bits, n, out, (cudaStream_t)stream), "log_det range");
  return SRT_OK;
}

srt_status srt_row_noise(int32_t vocab_size, uint64_t seed, int32_t n, const uint64_t* seq_id,
                         const int32_t* pos, float* out, void* stream) {
  if (vocab_size < 2 || n < 0 || (n > 0 && (!seq_id || !pos || !out))) return SRT_ERR_INVALID_ARG;
  if (n == 0) return SRT_OK;
  SRT_CUDA(launch_row_noise(vocab_size, seed, seq_id, pos, n, out, (cudaStream_t)stream),
           "row noise");
  return SRT_OK;
}

srt_status srt_stream_read(const void* buf, int64_t bytes, int32_t chunk, int32_t nbuf,
                           int32_t ctas_per_sm, void* sink, void* stream) {
  if (!buf || !sink || bytes < 0 || chunk < 1024 || chunk % 1024 || nbuf < 1 || ctas_per_sm < 1 ||
      (int64_t)nbuf * chunk * ctas_per_sm > 227 * 1024)
    return SRT_ERR_INVALID_ARG;
  SRT_CUDA(launch_stream_read(buf, bytes, chunk, nbuf, ctas_per_sm, (unsigned long long*)sink,
                              (cudaStream_t)stream),
           "stream read");
  return SRT_OK;
}

srt_status srt_cache_dump(srt_cache* c, int32_t p, srt_dump_record* host_buf, int64_t cap,
                          int64_t* n_records, void* stream_) {
  SRT_NVTX("srt_cache_dump");
  if (!c || !n_records || p < 0 || p >= c->cfg.max_prompts || cap < 0) return SRT_ERR_INVALID_ARG;
  cudaStream_t stream = (cudaStream_t)stream_;
  uint32_t bits = 0;
  srt_status st = srt_cache_status(c, &bits, nullptr, stream);
  if (st == SRT_ERR_CUDA) return st;
  if (bits & SRT_DEV_CAPACITY) return SRT_ERR_DEVICE;
  // Breadth-first enumeration, one level per launch (<= D levels); the host
  // then sorts siblings by token and emits the preorder.
  struct HNode { int32_t tok; uint32_t cnt; std::vector<int64_t> kids; };
  std::vector<HNode> nodes;
  uint32_t root_nchild = 0;
  const uint32_t root = (uint32_t)(c->dev.H + (uint64_t)p);
  SRT_CUDA(cudaMemcpyAsync(&root_nchild, &c->dev.rec[2 * (size_t)root].x, 4, cudaMemcpyDeviceToHost,
                           stream), "dump");
  SRT_CUDA(cudaStreamSynchronize(stream), "dump");
  nodes.push_back(HNode{-1, 0, {}});
  std::vector<uint32_t> frontier = {root};
  std::vector<int64_t> frontier_idx = {0};
  std::vector<uint32_t> frontier_nch = {root_nchild};
  while (!frontier.empty()) {
    uint64_t total = 0;
    for (uint32_t x : frontier_nch) total += x;
    if (total == 0) break;
    uint32_t *d_front = nullptr, *d_node = nullptr, *d_cnt = nullptr, *d_nch = nullptr;
    int32_t *d_par = nullptr, *d_tok = nullptr;
    unsigned int* d_n = nullptr;
    const int32_t nf = (int32_t)frontier.size();
    SRT_CUDA(cudaMallocAsync(&d_front, nf * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_node, total * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_cnt, total * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_nch, total * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_par, total * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_tok, total * 4, stream), "dump alloc");
    SRT_CUDA(cudaMallocAsync(&d_n, 4, stream), "dump alloc");
    SRT_CUDA(cudaMemsetAsync(d_n, 0, 4, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(d_front, frontier.data(), nf * 4, cudaMemcpyHostToDevice, stream), "dump");
    SRT_CUDA(launch_dump_level(c->dev, d_front, nf, d_node, d_par, d_tok, d_cnt, d_nch, d_n, stream),
             "dump kernel");
    std::vector<uint32_t> h_node(total), h_cnt(total), h_nch(total);
    std::vector<int32_t> h_par(total), h_tok(total);
    unsigned int h_n = 0;
    SRT_CUDA(cudaMemcpyAsync(&h_n, d_n, 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(h_node.data(), d_node, total * 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(h_cnt.data(), d_cnt, total * 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(h_nch.data(), d_nch, total * 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(h_par.data(), d_par, total * 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaMemcpyAsync(h_tok.data(), d_tok, total * 4, cudaMemcpyDeviceToHost, stream), "dump");
    SRT_CUDA(cudaStreamSynchronize(stream), "dump");
    cudaFreeAsync(d_front, stream); cudaFreeAsync(d_node, stream); cudaFreeAsync(d_cnt, stream);
    cudaFreeAsync(d_nch, stream); cudaFreeAsync(d_par, stream); cudaFreeAsync(d_tok, stream);
    cudaFreeAsync(d_n, stream);
    if (h_n != total) {
      snprintf(g_err, sizeof g_err, "dump: child count mismatch (%u vs %llu)", h_n,
               (unsigned long long)total);
      return SRT_ERR_CUDA;
    }
    std::vector<uint32_t> nf_nodes;
    std::vector<int64_t> nf_idx;
    std::vector<uint32_t> nf_nch;
    for (uint64_t k = 0; k < total; ++k) {
      int64_t idx = (int64_t)nodes.size();
      nodes.push_back(HNode{h_tok[k], h_cnt[k], {}});
      nodes[frontier_idx[h_par[k]]].kids.push_back(idx);
      nf_nodes.push_back(h_node[k]);
      nf_idx.push_back(idx);
      nf_nch.push_back(h_nch[k]);
    }
    frontier.swap(nf_nodes);
    frontier_idx.swap(nf_idx);
    frontier_nch.swap(nf_nch);
  }
  // preorder with children ascending by token
  int64_t k = 0;
  std::vector<int64_t> stack = {0};
  while (!stack.empty()) {
    int64_t i = stack.back();
    stack.pop_back();
    HNode& h = nodes[i];
    std::sort(h.kids.begin(), h.kids.end(),
              [&](int64_t a, int64_t b) { return nodes[a].tok < nodes[b].tok; });
    if (host_buf && k < cap) {
      uint64_t count = h.cnt;
      if (i == 0) {
        count = 0;
        for (int64_t kid : h.kids) count += nodes[kid].cnt;
      }
      host_buf[k] = srt_dump_record{h.tok, (int32_t)h.kids.size(), count};
    }
    ++k;
    for (auto it = h.kids.rbegin(); it != h.kids.rend(); ++it) stack.push_back(*it);
  }
  *n_records = k;
  return SRT_OK;
}

}  // extern "C"
