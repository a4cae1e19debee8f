// draft.cu — srt_draft: the batched draft kernel (one warp per sequence,
// draft.cuh) and the row offsets.
#include "draft.cuh"

namespace srt {

namespace {

__global__ void __launch_bounds__(DRAFT_WARPS * 32)
k_draft(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
        const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ seq_len,
        const int32_t* __restrict__ pos_base, const uint32_t* __restrict__ cursor, uint32_t tag,
        int32_t* __restrict__ match_len, int32_t* __restrict__ draft_len,
        int32_t* __restrict__ draft_tok,
        int32_t* __restrict__ draft_parent, int32_t* __restrict__ draft_depth,
        int32_t* __restrict__ draft_pos, uint64_t* __restrict__ draft_mask) {
  __shared__ unsigned long long masks[DRAFT_WARPS][64];  // ancestor-or-self masks (O9)
  __shared__ Ent merge_buf[DRAFT_WARPS][64];             // frontier merges
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * DRAFT_WARPS + w;
  if (s >= n) return;
  draft_seq(c, s, prompt_id, seq_tok, stride, seq_len, pos_base, cursor, tag, match_len, draft_len,
            draft_tok, draft_parent, draft_depth, draft_pos, draft_mask, masks[w], merge_buf[w],
            lane, nullptr);
}

constexpr int SCAN_THREADS = 1024;  // one pass for the usual n <= 1024

// row_offsets[s] = sum_{s' < s} (draft_len[s'] + 1)  (logits rows: root + nodes)
__global__ void __launch_bounds__(SCAN_THREADS)
k_row_offsets(int32_t n, const int32_t* __restrict__ draft_len, int64_t* __restrict__ row_offsets) {
  __shared__ long long warp_tot[SCAN_THREADS / 32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < n; base += SCAN_THREADS) {
    const int32_t s = base + threadIdx.x;
    const long long w = s < n ? (long long)draft_len[s] + 1 : 0;
    long long x = w;
    for (int o = 1; o < 32; o <<= 1) {
      long long yv = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += yv;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      long long tt = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        long long yv = __shfl_up_sync(0xffffffffu, tt, o);
        if (lane >= o) tt += yv;
      }
      if (lane < SCAN_THREADS / 32) warp_tot[lane] = tt;
    }
    __syncthreads();
    const long long before = carry + (wid ? warp_tot[wid - 1] : 0) + x - w;
    if (s < n) row_offsets[s] = before;
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry = before + w;
    __syncthreads();
  }
  if (threadIdx.x == 0) row_offsets[n] = carry;
}

}  // namespace

cudaError_t set_draft_profile(long long* buf) {
  return cudaMemcpyToSymbol(g_draft_prof, &buf, sizeof(buf));
}

cudaError_t launch_draft(const DevCache& c, int32_t n, const int32_t* prompt_id,
                         const int32_t* seq_tok, int64_t stride, const int32_t* seq_len,
                         const int32_t* pos_base, const uint32_t* cursor, uint32_t tag,
                         int32_t* match_len, int32_t* draft_len,
                         int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                         int32_t* draft_pos, uint64_t* draft_mask, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  carveout_once<k_draft>();
  k_draft<<<(n + DRAFT_WARPS - 1) / DRAFT_WARPS, DRAFT_WARPS * 32, 0, stream>>>(
      c, n, prompt_id, seq_tok, stride, seq_len, pos_base, cursor, tag, match_len, draft_len,
      draft_tok, draft_parent, draft_depth, draft_pos, draft_mask);
  return cudaGetLastError();
}

cudaError_t launch_row_offsets(int32_t n, const int32_t* draft_len, int64_t* row_offsets,
                               cudaStream_t stream) {
  carveout_once<k_row_offsets>();
  k_row_offsets<<<1, SCAN_THREADS, 0, stream>>>(n, draft_len, row_offsets);
  return cudaGetLastError();
}

}  // namespace srt
