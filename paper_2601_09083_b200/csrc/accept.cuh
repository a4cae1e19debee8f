// accept.cuh — the accept + commit walk of one sequence (one warp), shared by
// k_accept (verify.cu) and the fused accept + cursor insert (insert.cu).
// P:L46 (first mismatch, commit accepted tokens + one bonus token), DESIGN.md
// O10 / O13; EOS and length truncation as srt_verify documents (include/srt.h).
#pragma once
#include "srt_internal.cuh"

namespace srt {

// First decodes the scan's packed per-row winner into sampled[] (0 if the row
// had no candidate, i.e. every logit NaN, -1 for a row srt_verify_path did not
// sample), then walks the draft from its root and commits.  ctok: [Bmax + 1],
// acc: [Bmax] per-warp shared scratch.  Returns the sequence length before
// the commit (the committed span is [t, t + n_commit[s])).
__device__ __forceinline__ int32_t accept_seq(const DevCache& c, const VerifyArgs& a,
                                              const unsigned long long* __restrict__ result,
                                              int32_t s, int32_t* ctok, int32_t* acc, int lane) {
  const int32_t B = c.Bmax;
  const int32_t ns = a.draft_len[s];
  const int64_t r0 = a.row_offsets[s];
  for (int32_t i = lane; i <= ns; i += 32) {  // (~0: a row srt_verify_path did not sample)
    const unsigned long long rr = result[r0 + i];
    a.sampled[r0 + i] = rr == ~0ull ? -1 : unpack_index(rr);
  }
  __syncwarp();
  const int32_t t = a.seq_len[s];
  const int64_t db = (int64_t)s * B;
  const bool vA = lane < ns, vB = lane + 32 < ns;
  const int32_t tokA = vA ? a.draft_tok[db + lane] : -1;
  const int32_t parA = vA ? a.draft_parent[db + lane] : -2;
  const int32_t smpA = vA ? a.sampled[r0 + 1 + lane] : 0;
  const int32_t tokB = vB ? a.draft_tok[db + lane + 32] : -1;
  const int32_t parB = vB ? a.draft_parent[db + lane + 32] : -2;
  const int32_t smpB = vB ? a.sampled[r0 + 33 + lane] : 0;
  const int32_t root = a.sampled[r0];
  int32_t cur = -1, na = 0;
  while (true) {
    const int32_t sa = __shfl_sync(0xffffffffu, smpA, cur & 31);
    const int32_t sb = __shfl_sync(0xffffffffu, smpB, cur & 31);
    const int32_t tau = cur < 0 ? root : (cur < 32 ? sa : sb);
    if (lane == 0) ctok[na] = tau;
    const unsigned m0 = __ballot_sync(0xffffffffu, vA && parA == cur && tokA == tau);
    const unsigned m1 = __ballot_sync(0xffffffffu, vB && parB == cur && tokB == tau);
    const int32_t next = m0 ? __ffs(m0) - 1 : (m1 ? 31 + __ffs(m1) : -1);
    if (next < 0 || na >= B) break;
    if (lane == 0) acc[na] = next;
    ++na;
    cur = next;
  }
  __syncwarp();
  int32_t nc = na + 1;
  const int32_t cap = max(0, a.max_new[s] - t);
  nc = min(nc, cap);
  bool hit = false;
  if (a.eos_id >= 0) {
    int32_t first = INT_MAX;
    for (int32_t k = lane; k < nc; k += 32)
      if (ctok[k] == a.eos_id) first = min(first, k);
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (first != INT_MAX) { nc = first + 1; hit = true; }
  }
  for (int32_t k = lane; k < B + 1; k += 32) {
    const int32_t v = k < nc ? ctok[k] : -1;
    a.commit_tok[(int64_t)s * (B + 1) + k] = v;
    if (k < nc) a.seq_tok[(int64_t)s * a.stride + t + k] = v;
  }
  for (int32_t k = lane; k < B; k += 32) a.accepted_nodes[db + k] = k < na ? acc[k] : -1;
  if (lane == 0) {
    a.accept_len[s] = na;
    a.n_commit[s] = nc;
    a.seq_len[s] = t + nc;
    a.finished[s] = (hit || t + nc >= a.max_new[s]) ? 1 : 0;
  }
  return t;
}

}  // namespace srt
