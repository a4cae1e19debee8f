// draft.cu — srt_draft: batched longest-suffix match, best-first draft
// expansion and tree-attention layout (readings O3-O9).
//
// One warp per sequence.  Match: lane q-1 walks the root along y[t-q .. t-1]
// (q hash probes, all lanes in parallel) and a ballot keeps the largest q whose
// node has a child.  Expansion: a frontier sorted under the total order O8 is
// kept in shared memory (<= Bmax entries, truncated to B - popped, which is
// exact because a child never outranks its parent); the children of each
// popped node are enumerated 32 at a time from its child blocks (coalesced
// reads of the child ids and their token / count mirrors) and inserted with
// warp ballots.
// Roofline: latency-bound (L + ~3 B dependent loads per warp); us per batch.
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int DRAFT_WARPS = 2;  // 8K registers per CTA: fits beside a running verify scan

// Development-only per-sequence profile (srt_debug_draft_profile): when set,
// k_draft writes {match cycles, total cycles, children scanned, max children
// of one node, cycles in: record loads, block lookups, child loads,
// frontier inserts} per sequence.
__device__ long long* g_draft_prof = nullptr;
struct ExpandProf {
  long long rec = 0, blk = 0, ld = 0, ins = 0;
};
constexpr int FCAP = 64;

struct FrontierSmem {
  double score[FCAP];
  int32_t depth[FCAP];
  int32_t tok[FCAP];
  int32_t parent[FCAP];
  uint32_t node[FCAP];
  unsigned long long mask[FCAP];  // ancestor-or-self masks of drafted nodes
};

struct Cand {
  double score;
  int32_t depth, tok, parent;
  uint32_t node;
};

// O8: score desc, depth asc, token asc, parent draft index asc.
__device__ __forceinline__ bool better(double s1, int32_t d1, int32_t t1, int32_t p1, double s2,
                                       int32_t d2, int32_t t2, int32_t p2) {
  if (s1 != s2) return s1 > s2;
  if (d1 != d2) return d1 < d2;
  if (t1 != t2) return t1 < t2;
  return p1 < p2;
}

__device__ __forceinline__ bool entry_better(const FrontierSmem& F, int j, const Cand& c) {
  return better(F.score[j], F.depth[j], F.tok[j], F.parent[j], c.score, c.depth, c.tok, c.parent);
}

// Insert c into the sorted frontier of current size `size`, keeping at most
// `cap` entries.  Warp-collective; returns the new size.
__device__ __forceinline__ int frontier_insert(FrontierSmem& F, int size, int cap, const Cand& c,
                                               int lane) {
  const bool b0 = lane < size && entry_better(F, lane, c);
  const bool b1 = lane + 32 < size && entry_better(F, lane + 32, c);
  const int pos = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (pos >= cap) return size;
  const int newsize = min(size + 1, cap);
  Cand e0, e1;
  const bool m0 = lane >= pos && lane < newsize - 1;
  const bool m1 = lane + 32 >= pos && lane + 32 < newsize - 1;
  if (m0) e0 = Cand{F.score[lane], F.depth[lane], F.tok[lane], F.parent[lane], F.node[lane]};
  if (m1) e1 = Cand{F.score[lane + 32], F.depth[lane + 32], F.tok[lane + 32], F.parent[lane + 32],
                    F.node[lane + 32]};
  __syncwarp();
  if (m0) {
    F.score[lane + 1] = e0.score; F.depth[lane + 1] = e0.depth; F.tok[lane + 1] = e0.tok;
    F.parent[lane + 1] = e0.parent; F.node[lane + 1] = e0.node;
  }
  if (m1) {
    F.score[lane + 33] = e1.score; F.depth[lane + 33] = e1.depth; F.tok[lane + 33] = e1.tok;
    F.parent[lane + 33] = e1.parent; F.node[lane + 33] = e1.node;
  }
  __syncwarp();
  if (lane == 0) {
    F.score[pos] = c.score; F.depth[pos] = c.depth; F.tok[pos] = c.tok;
    F.parent[pos] = c.parent; F.node[pos] = c.node;
  }
  __syncwarp();
  return newsize;
}

__device__ __forceinline__ Cand frontier_pop(FrontierSmem& F, int size, int lane) {
  const Cand top{F.score[0], F.depth[0], F.tok[0], F.parent[0], F.node[0]};
  Cand e0, e1;
  const bool m0 = lane >= 1 && lane < size;
  const bool m1 = lane + 32 < size;
  if (m0) e0 = Cand{F.score[lane], F.depth[lane], F.tok[lane], F.parent[lane], F.node[lane]};
  if (m1) e1 = Cand{F.score[lane + 32], F.depth[lane + 32], F.tok[lane + 32], F.parent[lane + 32],
                    F.node[lane + 32]};
  __syncwarp();
  if (m0) {
    F.score[lane - 1] = e0.score; F.depth[lane - 1] = e0.depth; F.tok[lane - 1] = e0.tok;
    F.parent[lane - 1] = e0.parent; F.node[lane - 1] = e0.node;
  }
  if (m1) {
    F.score[lane + 31] = e1.score; F.depth[lane + 31] = e1.depth; F.tok[lane + 31] = e1.tok;
    F.parent[lane + 31] = e1.parent; F.node[lane + 31] = e1.node;
  }
  __syncwarp();
  return top;
}


// ---- register frontier (cap <= 32): lane i holds entry i while a node's
// children stream past, so each candidate costs one compare against the
// current bar (entry cap-1) and an entering one a ballot and a lane shift.
constexpr int32_t IMAX = 0x7FFFFFFF;
__device__ __forceinline__ Cand cand_shfl(const Cand& e, int src) {
  return Cand{__shfl_sync(0xffffffffu, e.score, src), __shfl_sync(0xffffffffu, e.depth, src),
              __shfl_sync(0xffffffffu, e.tok, src), __shfl_sync(0xffffffffu, e.parent, src),
              __shfl_sync(0xffffffffu, e.node, src)};
}
__device__ __forceinline__ Cand cand_shfl_up1(const Cand& e) {
  return Cand{__shfl_up_sync(0xffffffffu, e.score, 1), __shfl_up_sync(0xffffffffu, e.depth, 1),
              __shfl_up_sync(0xffffffffu, e.tok, 1), __shfl_up_sync(0xffffffffu, e.parent, 1),
              __shfl_up_sync(0xffffffffu, e.node, 1)};
}
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  return better(a.score, a.depth, a.tok, a.parent, b.score, b.depth, b.tok, b.parent);
}

// Push the children of u (C(v) = count(v) / csum(u), csum = the sum of the
// counts of u's children; score = score_u * C) into the
// frontier.  rec[u] is one 16-byte load; a single child needs nothing else
// (its C is exactly 1); more children are enumerated 32 x UNR at a time with
// every load of a round issued before any is used.
__device__ int expand(const DevCache& c, FrontierSmem& F, int size, int cap, uint32_t u,
                      double score_u, int32_t depth_u, int32_t parent_idx, int lane,
                      ExpandProf& pf) {
  if (cap <= 0) return size;
  long long t0 = clock64();
  const uint4 r = ld_rec(c, u);
  const uint32_t nch = r.x;
  pf.rec += clock64() - t0;
  if (nch == 0) return size;
  if (nch == 1) {
    // C = cnt(child0) / csum(u) = 1 exactly when csum > 0 (0/0 -> 0, O6)
    const Cand b{r.w ? __dmul_rn(score_u, 1.0) : 0.0, depth_u + 1, (int32_t)r.z, parent_idx, r.y};
    if (size == cap && !better(b.score, b.depth, b.tok, b.parent, F.score[cap - 1],
                               F.depth[cap - 1], F.tok[cap - 1], F.parent[cap - 1]))
      return size;
    return frontier_insert(F, size, cap, b, lane);
  }
  const double dsum = (double)r.w;  // exact (< 2^32)
  // block bases of blocks 0..nb-1 (children 1..nch-1), one lane each
  const uint32_t nb = blk_index(nch - 2) + 1;
  t0 = clock64();
  const uint32_t mybase = lane < (int)nb ? hash_find(c, block_key(u, lane)) : 0u;
  __syncwarp();
  pf.blk += clock64() - t0;
  constexpr int UNR = 8;
  if (cap <= 32) {
    const Cand SENT{-1.0, IMAX, IMAX, IMAX, NONE};  // worse than every real entry (scores >= 0)
    Cand fr = SENT;
    if (lane < size) fr = Cand{F.score[lane], F.depth[lane], F.tok[lane], F.parent[lane], F.node[lane]};
    Cand worst = cand_shfl(fr, cap - 1);  // the bar to enter
    for (uint32_t kr = 0; kr < nch; kr += 32 * UNR) {
      Cand cd[UNR];
      uint32_t cc[UNR];
      t0 = clock64();
#pragma unroll
      for (int m = 0; m < UNR; ++m) {  // child id, token and count mirror: coalesced
        const uint32_t k = kr + m * 32 + lane;
        const uint32_t jj = k >= 1 ? k - 1 : 0;
        const uint32_t bi = blk_index(jj);
        const uint32_t base = __shfl_sync(0xffffffffu, mybase, (int)(bi & 31));
        const uint32_t pos = base + (jj - blk_start(bi));
        cd[m] = Cand{-1.0, depth_u + 1, IMAX, parent_idx, NONE};
        cc[m] = 0;
        if (k == 0) {
          cd[m].node = r.y;
          cd[m].tok = (int32_t)r.z;
          cc[m] = __ldg(&c.cnt[r.y]);
        } else if (k < nch) {
          cd[m].node = __ldg(&c.slots[pos]);
          cd[m].tok = __ldg(&c.stok[pos]);
          cc[m] = __ldg(&c.scnt[pos]);
        }
      }
      __syncwarp();
      pf.ld += clock64() - t0;
      t0 = clock64();
#pragma unroll
      for (int m = 0; m < UNR; ++m)  // independent: the divisions pipeline
        if (cd[m].node != NONE)
          cd[m].score = __dmul_rn(score_u, r.w ? __ddiv_rn((double)cc[m], dsum) : 0.0);
#pragma unroll
      for (int m = 0; m < UNR; ++m) {
        if (kr + m * 32 >= nch) break;
        unsigned pending = __ballot_sync(0xffffffffu, cand_better(cd[m], worst));
        while (pending) {
          const int src = __ffs(pending) - 1;
          pending &= pending - 1;
          const Cand b = cand_shfl(cd[m], src);
          if (!cand_better(b, worst)) continue;  // an earlier insertion raised the bar
          const int at = __popc(__ballot_sync(0xffffffffu, cand_better(fr, b)));
          const Cand prev = cand_shfl_up1(fr);
          if (lane > at) fr = prev;
          if (lane == at) fr = b;
          worst = cand_shfl(fr, cap - 1);
        }
      }
      pf.ins += clock64() - t0;
    }
    const int nsize = __popc(__ballot_sync(0xffffffffu, lane < cap && fr.score >= 0.0));
    __syncwarp();
    if (lane < nsize) {
      F.score[lane] = fr.score; F.depth[lane] = fr.depth; F.tok[lane] = fr.tok;
      F.parent[lane] = fr.parent; F.node[lane] = fr.node;
    }
    __syncwarp();
    return nsize;
  }
  for (uint32_t kr = 0; kr < nch; kr += 32 * UNR) {
    uint32_t ch[UNR], cc[UNR];
    int32_t tk[UNR];
    t0 = clock64();
#pragma unroll
    for (int m = 0; m < UNR; ++m) {  // child id, token and count mirror: coalesced
      const uint32_t k = kr + m * 32 + lane;
      const uint32_t jj = k >= 1 ? k - 1 : 0;
      const uint32_t bi = blk_index(jj);
      const uint32_t base = __shfl_sync(0xffffffffu, mybase, (int)(bi & 31));
      const uint32_t pos = base + (jj - blk_start(bi));
      ch[m] = NONE;
      cc[m] = 0;
      tk[m] = 0;
      if (k == 0) {
        ch[m] = r.y;
        tk[m] = (int32_t)r.z;
        cc[m] = __ldg(&c.cnt[r.y]);
      } else if (k < nch) {
        ch[m] = __ldg(&c.slots[pos]);
        tk[m] = __ldg(&c.stok[pos]);
        cc[m] = __ldg(&c.scnt[pos]);
      }
    }
    __syncwarp();
    pf.ld += clock64() - t0;
    t0 = clock64();
#pragma unroll
    for (int m = 0; m < UNR; ++m) {
      if (kr + m * 32 >= nch) break;
      const bool valid = ch[m] != NONE;
      Cand cd{0.0, depth_u + 1, tk[m], parent_idx, ch[m]};
      if (valid) cd.score = __dmul_rn(score_u, r.w ? __ddiv_rn((double)cc[m], dsum) : 0.0);
      // cheap prefilter against the current worst entry when full
      bool want = valid;
      if (want && size == cap) want = !entry_better(F, cap - 1, cd);
      unsigned pending = __ballot_sync(0xffffffffu, want);
      while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        Cand b;
        b.score = __shfl_sync(0xffffffffu, cd.score, src);
        b.depth = cd.depth;
        b.tok = __shfl_sync(0xffffffffu, cd.tok, src);
        b.parent = parent_idx;
        b.node = __shfl_sync(0xffffffffu, cd.node, src);
        // re-check: earlier insertions of this round may have raised the worst entry
        if (size == cap && entry_better(F, cap - 1, b)) continue;
        size = frontier_insert(F, size, cap, b, lane);
      }
    }
    pf.ins += clock64() - t0;
  }
  return size;
}

__global__ void __launch_bounds__(DRAFT_WARPS * 32)
k_draft(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
        const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ seq_len,
        const int32_t* __restrict__ pos_base, int32_t* __restrict__ match_len,
        int32_t* __restrict__ draft_len, int32_t* __restrict__ draft_tok,
        int32_t* __restrict__ draft_parent, int32_t* __restrict__ draft_depth,
        int32_t* __restrict__ draft_pos, uint64_t* __restrict__ draft_mask) {
  __shared__ FrontierSmem smem[DRAFT_WARPS];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * DRAFT_WARPS + w;
  if (s >= n) return;
  FrontierSmem& F = smem[w];
  const long long t_start = clock64();
  long long t_match = 0, scanned = 0, maxch = 0;
  ExpandProf pf;
  const int32_t p = prompt_id[s];
  const int32_t t = seq_len[s];
  const int32_t* y = seq_tok + (int64_t)s * stride;
  const int32_t Bmax = c.Bmax;
  const int32_t pb = pos_base ? pos_base[s] : 0;
  int32_t q = 0;
  uint32_t uq = 0;
  if (p < 0 || p >= c.P) {
    if (lane == 0) set_error(c, SRT_DEV_BAD_PROMPT);
  } else {
    // ---- longest-suffix match (O3): lane handles q = lane + 1
    const int32_t qmax = min(c.L, t);
    const int32_t myq = lane + 1;
    bool ok = myq <= qmax;
    uint32_t node = (uint32_t)p;
    if (ok) {
      for (int32_t j = t - myq; j < t; ++j) {
        const int32_t tk = y[j];
        if (tk < 0 || tk >= c.V) {
          set_error(c, SRT_DEV_OOV);
          ok = false;
          break;
        }
        node = child_of(c, node, tk);
        if (node == NONE) {
          ok = false;
          break;
        }
      }
    }
    const bool has = ok && ld_rec(c, node).x > 0;
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    q = bal ? 32 - __clz(bal) : 0;
    uq = __shfl_sync(0xffffffffu, node, q > 0 ? q - 1 : 0);
  }
  t_match = clock64() - t_start;
  int32_t popped = 0;
  if (q > 0) {
    const long long bq = (long long)c.b0 + ((long long)q * c.snum) / c.sden;
    const int32_t B = (int32_t)min((long long)Bmax, bq);
    if (g_draft_prof) {
      const long long nc = ld_rec(c, uq).x;
      scanned += nc;
      maxch = max(maxch, nc);
    }
    int size = expand(c, F, 0, B, uq, 1.0, 0, -1, lane, pf);
    while (popped < B && size > 0) {
      __syncwarp();
      if (F.score[0] < c.min_score) break;
      const Cand top = frontier_pop(F, size, lane);
      --size;
      const int32_t i = popped++;
      if (lane == 0) {
        const unsigned long long m =
            (top.parent >= 0 ? F.mask[top.parent] : 0ull) | (1ull << i);
        F.mask[i] = m;
        const int64_t o = (int64_t)s * Bmax + i;
        draft_tok[o] = top.tok;
        draft_parent[o] = top.parent;
        draft_depth[o] = top.depth;
        draft_pos[o] = pb + top.depth;
        draft_mask[o] = m;
      }
      __syncwarp();
      const int cap = B - popped;
      if (size > cap) size = cap;
      if (g_draft_prof) {
        const long long nc = ld_rec(c, top.node).x;
        scanned += nc;
        maxch = max(maxch, nc);
      }
      size = expand(c, F, size, cap, top.node, top.score, top.depth, i, lane, pf);
    }
  }
  for (int32_t i = popped + lane; i < Bmax; i += 32) {
    const int64_t o = (int64_t)s * Bmax + i;
    draft_tok[o] = -1;
    draft_parent[o] = -1;
    draft_depth[o] = 0;
    draft_pos[o] = -1;
    draft_mask[o] = 0;
  }
  if (lane == 0) {
    match_len[s] = q;
    draft_len[s] = popped;
    if (g_draft_prof) {
      long long* o = g_draft_prof + 8 * (int64_t)s;
      o[0] = t_match;
      o[1] = clock64() - t_start;
      o[2] = scanned;
      o[3] = maxch;
      o[4] = pf.rec;
      o[5] = pf.blk;
      o[6] = pf.ld;
      o[7] = pf.ins;
    }
  }
}

constexpr int SCAN_THREADS = 256;  // small: co-resides with a running verify scan

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
                         const int32_t* pos_base, int32_t* match_len, int32_t* draft_len,
                         int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                         int32_t* draft_pos, uint64_t* draft_mask, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  carveout_once<k_draft>();
  k_draft<<<(n + DRAFT_WARPS - 1) / DRAFT_WARPS, DRAFT_WARPS * 32, 0, stream>>>(
      c, n, prompt_id, seq_tok, stride, seq_len, pos_base, match_len, draft_len, draft_tok,
      draft_parent, draft_depth, draft_pos, draft_mask);
  return cudaGetLastError();
}

cudaError_t launch_row_offsets(int32_t n, const int32_t* draft_len, int64_t* row_offsets,
                               cudaStream_t stream) {
  carveout_once<k_row_offsets>();
  k_row_offsets<<<1, SCAN_THREADS, 0, stream>>>(n, draft_len, row_offsets);
  return cudaGetLastError();
}

}  // namespace srt
