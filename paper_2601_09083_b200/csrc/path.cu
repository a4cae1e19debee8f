// path.cu — path-only verification (srt_verify_path).
//
// srt_verify samples the policy's token at EVERY draft row (the full scan
// reads every row once).  The commit only needs the rows on the accepted path
// (the root, each accepted node, and the row where the walk stops), so
// srt_verify_path walks level by level: round r scans one row per still-active
// sequence (its current node), then a step kernel finds the draft child whose
// token equals that row's sample and lists its row for round r + 1.  After R
// rounds the few sequences still accepting get their current node's whole
// draft subtree scanned at once, and k_accept finishes every walk exactly as
// in srt_verify.  Same commits, accepted lengths, sequence tables (the samples
// along the path are the same Gumbel-max draws, O11); rows off the path report
// sampled = -1.  No host synchronisation: row counts live on the device.
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr unsigned long long UNSCANNED = ~0ull;  // result word of a row not sampled

struct PathScratch {
  int32_t* list[2];
  int64_t* count;  // [2]
  int32_t* cur;      // per sequence: current draft node (-1 = root), -2 = walk over
};

__host__ __device__ inline size_t path_list_len(int32_t n, int32_t B) { return (size_t)n * (B + 1); }

__host__ __device__ inline PathScratch path_layout(void* base, int32_t n, int32_t B) {
  PathScratch S;
  char* b = (char*)base;
  S.count = (int64_t*)b;
  b += 64;
  S.list[0] = (int32_t*)b;
  b += path_list_len(n, B) * 4;
  S.list[1] = (int32_t*)b;
  b += path_list_len(n, B) * 4;
  S.cur = (int32_t*)b;
  return S;
}

__global__ void k_path_init(VerifyArgs a, unsigned long long* __restrict__ result,
                            int2* __restrict__ rowinfo, PathScratch S) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) {
    S.count[0] = a.n;
    S.count[1] = 0;
  }
  if (s >= a.n) return;
  const int64_t r0 = a.row_offsets[s];
  const int32_t ns = a.draft_len[s];
  for (int32_t i = 1; i <= ns; ++i) result[r0 + i] = UNSCANNED;
  result[r0] = 0;
  rowinfo[r0] = make_int2(s, a.seq_len[s]);
  S.list[0][s] = (int32_t)r0;
  S.cur[s] = -1;
}

// One warp per sequence: the sample of the current node's row picks the draft
// child to descend into; its row joins the next list (or the walk ends).
__global__ void __launch_bounds__(128)
k_path_step(VerifyArgs a, int32_t B, unsigned long long* __restrict__ result,
            int2* __restrict__ rowinfo, PathScratch S, int nxt) {
  const int lane = threadIdx.x & 31;
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= a.n) return;
  const int32_t c = S.cur[s];
  if (c < -1) return;
  const int64_t r0 = a.row_offsets[s];
  const int32_t ns = a.draft_len[s];
  const int32_t tau = unpack_index(result[r0 + 1 + c]);
  const int64_t db = (int64_t)s * B;
  const bool vA = lane < ns, vB = lane + 32 < ns;
  const unsigned m0 = __ballot_sync(0xffffffffu, vA && a.draft_parent[db + lane] == c &&
                                                     a.draft_tok[db + lane] == tau);
  const unsigned m1 = __ballot_sync(0xffffffffu, vB && a.draft_parent[db + lane + 32] == c &&
                                                     a.draft_tok[db + lane + 32] == tau);
  const int32_t j = m0 ? __ffs(m0) - 1 : (m1 ? 31 + __ffs(m1) : -1);
  if (lane != 0) return;
  if (j < 0) {
    S.cur[s] = -2;
    return;
  }
  S.cur[s] = j;
  const int64_t rj = r0 + 1 + j;
  result[rj] = 0;
  rowinfo[rj] = make_int2(s, a.seq_len[s] + a.draft_depth[db + j]);
  S.list[nxt][atomicAdd((unsigned long long*)&S.count[nxt], 1ull)] = (int32_t)rj;
}

// One warp per sequence still walking: every descendant of its current node
// (whose row is already listed) joins the list.
__global__ void __launch_bounds__(128)
k_path_tail(VerifyArgs a, int32_t B, unsigned long long* __restrict__ result,
            int2* __restrict__ rowinfo, PathScratch S, int nxt) {
  __shared__ unsigned long long desc_smem[4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= a.n) return;
  const int32_t c = S.cur[s];
  if (c < 0) return;  // walk over, or still at the root (then nothing was scanned: R = 0 case
                      // handled by listing every row below)
  const int64_t r0 = a.row_offsets[s];
  const int32_t ns = a.draft_len[s];
  const int64_t db = (int64_t)s * B;
  if (lane == 0) {
    unsigned long long d = 1ull << c;  // nodes whose ancestor-or-self is c (parents precede children)
    for (int32_t k = c + 1; k < ns; ++k) {
      const int32_t p = a.draft_parent[db + k];
      if (p >= 0 && (d >> p & 1)) d |= 1ull << k;
    }
    desc_smem[w] = d & ~(1ull << c);
  }
  __syncwarp();
  const unsigned long long d = desc_smem[w];
  for (int32_t k = lane; k < ns; k += 32) {
    if (!(d >> k & 1)) continue;
    const int64_t rk = r0 + 1 + k;
    result[rk] = 0;
    rowinfo[rk] = make_int2(s, a.seq_len[s] + a.draft_depth[db + k]);
    S.list[nxt][atomicAdd((unsigned long long*)&S.count[nxt], 1ull)] = (int32_t)rk;
  }
}

// R = 0: every row (root and nodes) of every sequence, as srt_verify.
__global__ void k_path_all(VerifyArgs a, int32_t B, unsigned long long* __restrict__ result,
                           int2* __restrict__ rowinfo, PathScratch S) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const int64_t r0 = a.row_offsets[s];
  const int32_t ns = a.draft_len[s];
  for (int32_t k = 0; k < ns; ++k) {
    const int64_t rk = r0 + 1 + k;
    result[rk] = 0;
    rowinfo[rk] = make_int2(s, a.seq_len[s] + a.draft_depth[(int64_t)s * B + k]);
    S.list[0][atomicAdd((unsigned long long*)&S.count[0], 1ull)] = (int32_t)rk;
  }
}

}  // namespace

size_t path_scratch_bytes(int32_t n, int32_t B) { return 64 + 2 * path_list_len(n, B) * 4 + (size_t)n * 4 + 64; }

cudaError_t launch_path_verify(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                               unsigned long long* result, void* scratch, int rounds,
                               cudaStream_t stream) {
  const PathScratch S = path_layout(scratch, a.n, c.Bmax);
  const int tb = 128, wb = (a.n * 32 + tb - 1) / tb;
  k_path_init<<<(a.n + tb - 1) / tb, tb, 0, stream>>>(a, result, rowinfo, S);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int cur = 0;
  if (rounds <= 0) {
    k_path_all<<<(a.n + tb - 1) / tb, tb, 0, stream>>>(a, c.Bmax, result, rowinfo, S);
  } else {
    for (int r = 0; r < rounds; ++r) {
      if ((e = launch_scan_list(c, a, rowinfo, S.list[cur], S.count + cur, result, stream)) !=
          cudaSuccess)
        return e;
      if ((e = cudaMemsetAsync(S.count + (cur ^ 1), 0, 8, stream)) != cudaSuccess) return e;
      k_path_step<<<wb, tb, 0, stream>>>(a, c.Bmax, result, rowinfo, S, cur ^ 1);
      cur ^= 1;
    }
    k_path_tail<<<wb, tb, 0, stream>>>(a, c.Bmax, result, rowinfo, S, cur);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_scan_list(c, a, rowinfo, S.list[cur], S.count + cur, result, stream);
}

}  // namespace srt
