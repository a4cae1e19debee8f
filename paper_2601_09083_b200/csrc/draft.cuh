// draft.cuh — the draft of one sequence by one warp (srt_draft; step.cu): batched longest-suffix match, best-first draft
// expansion and tree-attention layout (readings O3-O9).
//
// One warp per sequence.  Match: lane q-1 walks the root along y[t-q .. t-1]
// (q hash probes, all lanes in parallel) and a ballot keeps the largest q whose
// node has a child.  Expansion: the frontier lives in registers, sorted under
// the total order O8 (lane i holds entries i and i + 32, so up to 64 entries),
// truncated to B - popped (exact: a child never outranks its parent).  A pop is
// a lane shift; a candidate enters with two ballots and a shift.  Children of
// a multi-child node stream past 32 x UNR at a time (coalesced child ids,
// tokens and count mirrors), the next round's loads in flight while this one
// is ranked, and a count threshold (the largest count whose score is below the
// frontier's last entry) rejects most of a hub's children with one integer
// compare before any division.
// Roofline: latency-bound (L probes + ~1 record load per pop + 1-2 round trips
// per multi-child pop per warp); us per batch.
#pragma once
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int DRAFT_WARPS = 2;  // small CTAs: fit beside a running verify scan

// Development-only per-sequence profile (srt_debug_draft_profile): when set,
// k_draft writes {match cycles, total cycles, children scanned, max children
// of one node, cycles waiting for records, cycles in block lookups, cycles in
// child rounds, (multi-child pops << 20) | single-child pops} per sequence.
__device__ long long* g_draft_prof = nullptr;
struct ExpandProf {
  long long rec = 0, blk = 0, ld = 0, pops = 0;
};

constexpr int32_t IMAX = 0x7FFFFFFF;
constexpr unsigned long long META_NONE = ~0ull;

// A frontier entry.  O8 orders entries by score desc, then depth asc, token
// asc, parent draft index asc; the last three are packed into `meta` so that a
// smaller meta is the better entry on equal scores:
//   meta = depth << 38 | token << 7 | (parent + 1)   (depth <= 64, token < 2^31,
//                                                     parent in [-1, 63])
struct Ent {
  double score;
  unsigned long long meta;
  uint32_t node;
};
__device__ __forceinline__ unsigned long long make_meta(int32_t depth, int32_t tok, int32_t parent) {
  return ((unsigned long long)depth << 38) | ((unsigned long long)(uint32_t)tok << 7) |
         (unsigned long long)(parent + 1);
}
__device__ __forceinline__ int32_t meta_depth(unsigned long long m) { return (int32_t)(m >> 38); }
__device__ __forceinline__ int32_t meta_tok(unsigned long long m) {
  return (int32_t)((m >> 7) & 0x7FFFFFFFull);
}
__device__ __forceinline__ int32_t meta_parent(unsigned long long m) { return (int32_t)(m & 0x7F) - 1; }

__device__ __forceinline__ bool better(const Ent& a, const Ent& b) {
  return a.score > b.score || (a.score == b.score && a.meta < b.meta);
}
__device__ __forceinline__ Ent ent_shfl(const Ent& e, int src) {
  return Ent{__shfl_sync(0xffffffffu, e.score, src), __shfl_sync(0xffffffffu, e.meta, src),
             __shfl_sync(0xffffffffu, e.node, src)};
}
__device__ __forceinline__ Ent ent_up1(const Ent& e) {
  return Ent{__shfl_up_sync(0xffffffffu, e.score, 1), __shfl_up_sync(0xffffffffu, e.meta, 1),
             __shfl_up_sync(0xffffffffu, e.node, 1)};
}
__device__ __forceinline__ Ent ent_down1(const Ent& e) {
  return Ent{__shfl_down_sync(0xffffffffu, e.score, 1), __shfl_down_sync(0xffffffffu, e.meta, 1),
             __shfl_down_sync(0xffffffffu, e.node, 1)};
}

// Loads the compiler may not sink to their first use (software pipelining of
// the child rounds) and fire-and-forget L1 prefetches.
__device__ __forceinline__ uint32_t ldg_early(const uint32_t* p) {
  uint32_t v;
#ifdef SRT_COHERENT_LOADS
  asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
#else
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// The register frontier: entry j on lane j (e0) or lane j - 32 (e1); entries
// [0, size) are valid and sorted, size <= cap <= 64.
struct Frontier {
  Ent e0, e1;
  int size;

  __device__ __forceinline__ Ent at(int j) const {
    return j < 32 ? ent_shfl(e0, j) : ent_shfl(e1, j - 32);
  }
  // Insert candidate b (warp-uniform); entries past cap fall off.
  __device__ __forceinline__ void insert(const Ent& b, int cap, int lane) {
    int pos = __popc(__ballot_sync(0xffffffffu, lane < size && better(e0, b)));
    if (size > 32) pos += __popc(__ballot_sync(0xffffffffu, lane + 32 < size && better(e1, b)));
    if (pos >= cap) return;
    const Ent u0 = ent_up1(e0);
    if (cap > 32) {  // (warp-uniform) entries 32.. live in e1
      const Ent u1 = ent_up1(e1);
      const Ent last0 = ent_shfl(e0, 31);
      if (lane + 32 >= pos) e1 = (lane + 32 == pos) ? b : (lane == 0 ? last0 : u1);
    }
    if (lane >= pos) e0 = (lane == pos) ? b : u0;
    size = min(size + 1, cap);
  }
  // Merge na sorted candidates (lane k holds candidate k, best first) into the
  // frontier in one pass: the result is the top cap of both, exactly what na
  // inserts in order would leave.  Each side's position in the merged order
  // is its index plus its rank in the other side (branchless binary searches
  // over shuffles); the merged entries are exchanged through sm (64 entries).
  // Returns whether the last candidate made it (if not, later ones cannot).
  __device__ __forceinline__ bool merge(const Ent& a, int na, int cap, int lane, Ent* sm) {
    const bool wide = cap > 32;  // (warp-uniform) entries 32.. in e1
    int ra = 0;                  // frontier entries better than a
    for (int step = wide ? 64 : 32; step >= 1; step >>= 1) {
      const int probe = ra + step - 1;
      const int src = probe & 31;
      const double s0 = __shfl_sync(0xffffffffu, e0.score, src);
      const unsigned long long m0 = __shfl_sync(0xffffffffu, e0.meta, src);
      double sc = s0;
      unsigned long long mt = m0;
      if (wide) {
        const double s1 = __shfl_sync(0xffffffffu, e1.score, src);
        const unsigned long long m1 = __shfl_sync(0xffffffffu, e1.meta, src);
        if (probe >= 32) { sc = s1; mt = m1; }
      }
      if (probe < size && better(Ent{sc, mt, 0u}, a)) ra += step;
    }
    int rb0 = 0, rb1 = 0;  // candidates better than frontier entries lane, lane + 32
    for (int step = 32; step >= 1; step >>= 1) {
      const int probe0 = rb0 + step - 1, probe1 = rb1 + step - 1;
      const double s0 = __shfl_sync(0xffffffffu, a.score, probe0 & 31);
      const unsigned long long m0 = __shfl_sync(0xffffffffu, a.meta, probe0 & 31);
      if (probe0 < na && better(Ent{s0, m0, 0u}, e0)) rb0 += step;
      if (wide) {
        const double s1 = __shfl_sync(0xffffffffu, a.score, probe1 & 31);
        const unsigned long long m1 = __shfl_sync(0xffffffffu, a.meta, probe1 & 31);
        if (probe1 < na && better(Ent{s1, m1, 0u}, e1)) rb1 += step;
      }
    }
    const int pa = lane + ra, p0 = lane + rb0, p1 = lane + 32 + rb1;
    if (lane < na && pa < cap) sm[pa] = a;
    if (lane < size && p0 < cap) sm[p0] = e0;
    if (wide && lane + 32 < size && p1 < cap) sm[p1] = e1;
    __syncwarp();
    const bool last_in = __shfl_sync(0xffffffffu, pa, (na - 1) & 31) < cap;
    size = min(size + na, cap);
    const Ent none{-1.0, META_NONE, NONE};
    e0 = lane < size ? sm[lane] : none;
    if (wide) e1 = lane + 32 < size ? sm[lane + 32] : none;
    __syncwarp();
    return last_in;
  }
  // Remove entry 0 (returned).
  __device__ __forceinline__ Ent pop(int lane) {
    const Ent top = ent_shfl(e0, 0);
    const Ent d0 = ent_down1(e0);
    if (size > 32) {  // (warp-uniform)
      const Ent d1 = ent_down1(e1);
      const Ent first1 = ent_shfl(e1, 0);
      e0 = lane < 31 ? d0 : first1;
      e1 = d1;
    } else {
      e0 = d0;
    }
    --size;
    return top;
  }
};

// f(c) = score of a child with count c (O6): RN(score_u * RN(c / csum)).
__device__ __forceinline__ double child_score(double score_u, double dsum, uint32_t c) {
  return __dmul_rn(score_u, dsum > 0.0 ? __ddiv_rn((double)c, dsum) : 0.0);
}

// A count c_lo such that every child with count <= c_lo scores strictly
// below w (so it cannot enter a full frontier whose last entry scores w), or
// -1.  One rounded estimate x' of x = w * csum / score_u has relative error
// below 2^-50, so floor(x') - 2 <= x - 1, and f(c) = RN(score_u * RN(c/csum))
// <= score_u * (x - 1) / csum * (1 + 2^-51) < w for every c <= x - 1 as long
// as x < 2^50 (counts < 2^32).  Exactness never depends on c_lo being tight.
__device__ __forceinline__ long long count_floor(double w, double score_u, double dsum) {
  if (!(w > 0.0) || score_u == 0.0) return -1;
  const double x = __ddiv_rn(__dmul_rn(w, dsum), score_u);
  if (!(x < 4294967296.0)) return (long long)dsum;  // every count scores below w
  return (long long)floor(x) - 2;
}

// Push the children of u (C(v) = count(v) / csum(u), csum = the sum of the
// counts of u's children; score = score_u * C) into the
// frontier.  rec[u] is one 16-byte load; a single child needs nothing else
// (its C is exactly 1).
__device__ void expand(const DevCache& c, Frontier& F, int cap, uint32_t u, double score_u,
                       int32_t depth_u, int32_t parent_idx, int lane, ExpandProf& pf, Ent* sm,
                       int32_t p, uint32_t* pdl) {
  if (cap <= 0) return;
  long long t0 = clock64();
  const uint4 r = ld_rec(c, u);
  uint32_t nch;
  asm volatile("mov.b32 %0, %1;" : "=r"(nch) : "r"(r.x));  // (profile: time the wait)
  pf.rec += clock64() - t0;
  if (nch == 0) return;
  if (nch == 1) {
    // C = cnt(child0) / csum(u) = 1 exactly when csum > 0 (0/0 -> 0, O6)
    ++pf.pops;
    F.insert(Ent{r.w ? score_u : 0.0, make_meta(depth_u + 1, (int32_t)r.z, parent_idx), r.y}, cap,
             lane);
    return;
  }
  pf.pops += 1ll << 20;
  const double dsum = (double)r.w;  // exact (< 2^32)
  const unsigned long long meta0 = make_meta(depth_u + 1, 0, parent_idx);
  if (nch > HUB_MIN && dsum > 0.0 && score_u > 1e-250) {
    // (a normal, nonzero score_u keeps the sibling score strictly increasing
    // in the count, so the list's order is the O8 order)
    // a hub: its top children by (count desc, token asc) are listed while its
    // child count and csum are unchanged (hub.cu); siblings rank by exactly
    // that order (O6, O8), so the first cap of them are all that can enter
    const uint32_t slot = hub_slot(c, p, u);
    const bool ok = SRT_LD(c.hub_node[slot]) == u && SRT_LD(c.hub_nch[slot]) == nch &&
                    SRT_LD(c.hub_csum[slot]) == r.w;
    if (ok) {
      const uint32_t len = min(SRT_LD(c.hub_len[slot]), (uint32_t)cap);
      const size_t e = (size_t)slot * HUB_K;
      for (uint32_t kb = 0; kb < len; kb += 32) {
        const uint32_t k = kb + lane;
        Ent cd{-1.0, META_NONE, NONE};
        if (k < len) {
          cd.node = SRT_LD(c.hub_child[e + k]);
          cd.score = child_score(score_u, dsum, SRT_LD(c.hub_cnt[e + k]));
          cd.meta = meta0 | ((unsigned long long)(uint32_t)SRT_LD(c.hub_tok[e + k]) << 7);
        }
        // candidates (sorted) that beat the current last entry: only they can enter
        const Ent bar = F.size == cap ? F.at(cap - 1) : Ent{-1.0, META_NONE, NONE};
        const int nb = __popc(__ballot_sync(0xffffffffu, k < len && better(cd, bar)));
        if (nb > 4) {  // many: one merge
          if (!F.merge(cd, nb, cap, lane, sm)) break;
        } else {  // few: inserts in order, stopping at the first loser
          bool stop = false;
          for (int src = 0; src < nb; ++src) {
            const Ent b = ent_shfl(cd, src);
            const Ent bar2 = F.size == cap ? F.at(cap - 1) : Ent{-1.0, META_NONE, NONE};
            if (!better(b, bar2)) {
              stop = true;
              break;
            }
            F.insert(b, cap, lane);
          }
          if (stop) break;
        }
        if (nb < 32) break;  // the rest of the list does not beat the last entry either
      }
      return;
    }
    if (lane == 0) {  // no valid list for this hub: the refresh after the next insert builds it
      if (pdl) {  // (the fused tree step: prompt p's own list)
        const uint32_t e = atomicAdd(pdl, 1u);
        if (e < PDIRTY_CAP) {  // (child NONE: rebuild from all children)
          pdl[2 + 2 * e] = u;
          pdl[3 + 2 * e] = NONE;
        }
      } else {
        const uint32_t e = atomicAdd(c.dirty_n, 1u);
        if (e < DIRTY_CAP) c.dirty[e] = make_uint2(u, (uint32_t)p);
      }
    }
  }
  // block bases of blocks 0..nb-1 (children 1..nch-1), one lane each
  const uint32_t nb = blk_index(nch - 2) + 1;
  t0 = clock64();
  const uint32_t mybase = lane < (int)nb ? block_base(c, u, lane) : 0u;
  __syncwarp();
  pf.blk += clock64() - t0;
  t0 = clock64();
  // the entry a candidate must beat, and the count at or below which none can
  Ent bar = F.size == cap ? F.at(cap - 1) : Ent{-1.0, META_NONE, NONE};
  long long c_lo = count_floor(bar.score, score_u, dsum);
  constexpr int UNR = 8;
  uint32_t chA[UNR], ccA[UNR], chB[UNR], ccB[UNR];
  int32_t tkA[UNR], tkB[UNR];
  auto load_round = [&](uint32_t kr, uint32_t (&ch)[UNR], int32_t (&tk)[UNR],
                        uint32_t (&cc)[UNR]) {
#pragma unroll
    for (int m = 0; m < UNR; ++m) {  // child id, token and count mirror: coalesced
      const uint32_t k = kr + m * 32 + lane;
      ch[m] = NONE;
      cc[m] = 0;
      tk[m] = IMAX;
      if (kr + m * 32 >= nch) continue;  // (warp-uniform)
      const uint32_t jj = k >= 1 ? k - 1 : 0;
      const uint32_t bi = blk_index(jj);
      const uint32_t base = __shfl_sync(0xffffffffu, mybase, (int)(bi & 31));
      const uint32_t pos = base + (jj - blk_start(bi));
      if (k == 0) {
        ch[m] = r.y;
        tk[m] = (int32_t)r.z;
        cc[m] = ldg_early(&c.cnt[r.y]);
      } else if (k < nch) {
        ch[m] = ldg_early(&c.slots[pos]);
        tk[m] = (int32_t)ldg_early((const uint32_t*)&c.stok[pos]);
        cc[m] = ldg_early(&c.scnt[pos]);
      }
    }
  };
  auto rank_round = [&](uint32_t kr, const uint32_t (&ch)[UNR], const int32_t (&tk)[UNR],
                        const uint32_t (&cc)[UNR]) {
    bool entered = false;
#pragma unroll
    for (int m = 0; m < UNR; ++m) {
      if (kr + m * 32 >= nch) break;
      // count prefilter, then the exact comparison against the bar
      Ent cd{-1.0, META_NONE, ch[m]};
      bool want = ch[m] != NONE && (long long)cc[m] > c_lo;
      if (want) {
        cd.score = child_score(score_u, dsum, cc[m]);
        cd.meta = meta0 | ((unsigned long long)(uint32_t)tk[m] << 7);
        want = better(cd, bar);
      }
      unsigned pending = __ballot_sync(0xffffffffu, want);
      while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const Ent b = ent_shfl(cd, src);
        if (!better(b, bar)) continue;  // an earlier insertion raised the bar
        F.insert(b, cap, lane);
        entered = true;
        if (F.size == cap) bar = F.at(cap - 1);
      }
    }
    if (entered && F.size == cap) c_lo = count_floor(bar.score, score_u, dsum);
  };
  load_round(0, chA, tkA, ccA);
  for (uint32_t kr = 0; kr < nch; kr += 64 * UNR) {
    const uint32_t k1 = kr + 32 * UNR;
    if (k1 < nch) load_round(k1, chB, tkB, ccB);
    rank_round(kr, chA, tkA, ccA);
    if (k1 >= nch) break;
    if (k1 + 32 * UNR < nch) load_round(k1 + 32 * UNR, chA, tkA, ccA);
    rank_round(k1, chB, tkB, ccB);
  }
  pf.ld += clock64() - t0;
}

// Warm L1 with what popping the next frontier entries reads first: their
// 32-byte records (child count, first child, csum and the first child blocks).
__device__ __forceinline__ void prefetch_frontier(const DevCache& c, const Frontier& F, int lane) {
  if (lane < 4 && lane < F.size) prefetch_l1(rec_of(c, F.e0.node));
}

// The draft of sequence s by one warp (O3-O9): match, best-first
// expansion, layout.  M: [64] ancestor masks and merge_buf: [64] frontier
// merge scratch of this warp in shared memory; pdl: null (hubs without a
// valid list go to the global dirty list) or prompt p's list (step.cu).
__device__ void draft_seq(const DevCache& c, int32_t s, const int32_t* __restrict__ prompt_id,
                          const int32_t* __restrict__ seq_tok, int64_t stride,
                          const int32_t* __restrict__ seq_len, const int32_t* __restrict__ pos_base,
                          const uint32_t* __restrict__ cursor, uint32_t tag,
                          int32_t* __restrict__ match_len, int32_t* __restrict__ draft_len,
                          int32_t* __restrict__ draft_tok, int32_t* __restrict__ draft_parent,
                          int32_t* __restrict__ draft_depth, int32_t* __restrict__ draft_pos,
                          uint64_t* __restrict__ draft_mask, unsigned long long* M, Ent* merge_buf,
                          int lane, uint32_t* pdirty) {
  long long* const prof = g_draft_prof;  // (development profile; one load)
  const long long t_start = clock64();
  long long t_match = 0, scanned = 0, maxch = 0;
  ExpandProf pf;
  const int32_t p = prompt_id[s];
  uint32_t* const pdl = (pdirty && p >= 0 && p < c.P) ? pdirty + (size_t)p * PDIRTY_WORDS : nullptr;
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
    uint32_t node = root_id(c, p);
    // a valid cursor at t with floor 0 holds node(y[t-q .. t-1]) for every
    // q <= min(D, t) (L <= D): no walk
    bool walk = true;
    if (cursor) {
      const uint32_t* cur = cursor + (size_t)s * (c.D + 4);
      if (cur[0] == tag && cur[1] == (uint32_t)t && cur[2] == (uint32_t)p && cur[3] == 0u) {
        walk = false;
        if (ok) {
          node = cur[4 + myq - 1];
          ok = node < BAD;
        }
      }
    }
    if (ok && walk) {
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
    if (prof) {
      const long long nc = ld_rec(c, uq).x;
      scanned += nc;
      maxch = max(maxch, nc);
    }
    Frontier F{Ent{-1.0, META_NONE, NONE}, Ent{-1.0, META_NONE, NONE}, 0};
    expand(c, F, B, uq, 1.0, 0, -1, lane, pf, merge_buf, p, pdl);
    prefetch_frontier(c, F, lane);
    while (popped < B && F.size > 0) {
      if (__shfl_sync(0xffffffffu, F.e0.score, 0) < c.min_score) break;
      const Ent top = F.pop(lane);
      const int32_t i = popped++;
      const int32_t par = meta_parent(top.meta), dep = meta_depth(top.meta);
      if (lane == 0) {
        const unsigned long long m = (par >= 0 ? M[par] : 0ull) | (1ull << i);
        M[i] = m;
        const int64_t o = (int64_t)s * Bmax + i;
        draft_tok[o] = meta_tok(top.meta);
        draft_parent[o] = par;
        draft_depth[o] = dep;
        draft_pos[o] = pb + dep;
        draft_mask[o] = m;
      }
      const int cap = B - popped;
      if (F.size > cap) F.size = cap;
      if (prof) {
        const long long nc = ld_rec(c, top.node).x;
        scanned += nc;
        maxch = max(maxch, nc);
      }
      expand(c, F, cap, top.node, top.score, dep, i, lane, pf, merge_buf, p, pdl);
      prefetch_frontier(c, F, lane);
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
    if (prof) {
      long long* o = prof + 8 * (int64_t)s;
      o[0] = t_match;
      o[1] = clock64() - t_start;
      o[2] = scanned;
      o[3] = maxch;
      o[4] = pf.rec;
      o[5] = pf.blk;
      o[6] = pf.ld;
      o[7] = pf.pops;
    }
  }
}


}  // namespace
}  // namespace srt
