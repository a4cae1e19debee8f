// exchange.cu — fixed-size draft / span records for the multi-GPU exchange
// (BJ:north_star: prompts hash-sharded over the GPUs, decoded spans
// all-gathered before insertion).  Pure data movement: one warp
// per record, coalesced along the record's words.
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int XW = 4;  // warps per CTA

__global__ void __launch_bounds__(XW * 32)
k_pack_drafts(int32_t n, int32_t B, const int32_t* __restrict__ match_len,
              const int32_t* __restrict__ draft_len, const int32_t* __restrict__ draft_tok,
              const int32_t* __restrict__ draft_parent, const int32_t* __restrict__ draft_depth,
              const uint64_t* __restrict__ draft_mask, int32_t* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int32_t s = blockIdx.x * XW + (threadIdx.x >> 5);
  if (s >= n) return;
  int32_t* r = rec + (int64_t)s * (2 + 5 * B);
  const int64_t o = (int64_t)s * B;
  if (lane == 0) {
    r[0] = match_len[s];
    r[1] = draft_len[s];
  }
  for (int32_t i = lane; i < B; i += 32) {
    r[2 + i] = draft_tok[o + i];
    r[2 + B + i] = draft_parent[o + i];
    r[2 + 2 * B + i] = draft_depth[o + i];
    const uint64_t m = draft_mask[o + i];
    r[2 + 3 * B + i] = (int32_t)(uint32_t)m;
    r[2 + 4 * B + i] = (int32_t)(uint32_t)(m >> 32);
  }
}

__global__ void __launch_bounds__(XW * 32)
k_unpack_drafts(int32_t n, int32_t B, const int32_t* __restrict__ rec,
                const int32_t* __restrict__ src, const int32_t* __restrict__ pos_base,
                int32_t* __restrict__ match_len, int32_t* __restrict__ draft_len,
                int32_t* __restrict__ draft_tok, int32_t* __restrict__ draft_parent,
                int32_t* __restrict__ draft_depth, int32_t* __restrict__ draft_pos,
                uint64_t* __restrict__ draft_mask) {
  const int lane = threadIdx.x & 31;
  const int32_t s = blockIdx.x * XW + (threadIdx.x >> 5);
  if (s >= n) return;
  const int32_t* r = rec + (int64_t)src[s] * (2 + 5 * B);
  const int64_t o = (int64_t)s * B;
  const int32_t len = r[1];
  const int32_t pb = pos_base ? pos_base[s] : 0;
  if (lane == 0) {
    match_len[s] = r[0];
    draft_len[s] = len;
  }
  for (int32_t i = lane; i < B; i += 32) {
    const int32_t d = r[2 + 2 * B + i];
    draft_tok[o + i] = r[2 + i];
    draft_parent[o + i] = r[2 + B + i];
    draft_depth[o + i] = d;
    draft_pos[o + i] = i < len ? pb + d : -1;
    draft_mask[o + i] = (uint64_t)(uint32_t)r[2 + 3 * B + i] |
                        ((uint64_t)(uint32_t)r[2 + 4 * B + i] << 32);
  }
}

__global__ void __launch_bounds__(XW * 32)
k_pack_spans(int32_t n, int32_t B, const int32_t* __restrict__ n_commit,
             const int32_t* __restrict__ commit_tok, int32_t* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int32_t s = blockIdx.x * XW + (threadIdx.x >> 5);
  if (s >= n) return;
  int32_t* r = rec + (int64_t)s * (B + 2);
  if (lane == 0) r[0] = n_commit[s];
  for (int32_t i = lane; i <= B; i += 32) r[1 + i] = commit_tok[(int64_t)s * (B + 1) + i];
}

__global__ void __launch_bounds__(XW * 32)
k_apply_spans(int32_t n, int32_t B, const int32_t* __restrict__ rec,
              const int32_t* __restrict__ src, int32_t* __restrict__ seq_tok, int64_t stride,
              int32_t* __restrict__ seq_len, int32_t* __restrict__ from, int32_t* __restrict__ to) {
  const int lane = threadIdx.x & 31;
  const int32_t m = blockIdx.x * XW + (threadIdx.x >> 5);
  if (m >= n) return;
  const int32_t* r = rec + (int64_t)src[m] * (B + 2);
  const int32_t t = seq_len[m];
  int32_t k = min(max(r[0], 0), B + 1);
  if ((int64_t)t + k > stride) k = stride > t ? (int32_t)(stride - t) : 0;
  for (int32_t i = lane; i < k; i += 32) seq_tok[(int64_t)m * stride + t + i] = r[1 + i];
  if (lane == 0) {
    from[m] = t;
    to[m] = t + k;
    seq_len[m] = t + k;
  }
}

inline int grid(int32_t n) { return (n + XW - 1) / XW; }

}  // namespace

cudaError_t launch_pack_drafts(int32_t n, int32_t B, const int32_t* match_len,
                               const int32_t* draft_len, const int32_t* draft_tok,
                               const int32_t* draft_parent, const int32_t* draft_depth,
                               const uint64_t* draft_mask, int32_t* rec, cudaStream_t stream) {
  k_pack_drafts<<<grid(n), XW * 32, 0, stream>>>(n, B, match_len, draft_len, draft_tok,
                                                  draft_parent, draft_depth, draft_mask, rec);
  return cudaGetLastError();
}

cudaError_t launch_unpack_drafts(int32_t n, int32_t B, const int32_t* rec, const int32_t* src,
                                 const int32_t* pos_base, int32_t* match_len, int32_t* draft_len,
                                 int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                                 int32_t* draft_pos, uint64_t* draft_mask, cudaStream_t stream) {
  k_unpack_drafts<<<grid(n), XW * 32, 0, stream>>>(n, B, rec, src, pos_base, match_len, draft_len,
                                                    draft_tok, draft_parent, draft_depth,
                                                    draft_pos, draft_mask);
  return cudaGetLastError();
}

cudaError_t launch_pack_spans(int32_t n, int32_t B, const int32_t* n_commit,
                              const int32_t* commit_tok, int32_t* rec, cudaStream_t stream) {
  k_pack_spans<<<grid(n), XW * 32, 0, stream>>>(n, B, n_commit, commit_tok, rec);
  return cudaGetLastError();
}

cudaError_t launch_apply_spans(int32_t n, int32_t B, const int32_t* rec, const int32_t* src,
                               int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* from,
                               int32_t* to, cudaStream_t stream) {
  k_apply_spans<<<grid(n), XW * 32, 0, stream>>>(n, B, rec, src, seq_tok, stride, seq_len, from,
                                                  to);
  return cudaGetLastError();
}

}  // namespace srt
