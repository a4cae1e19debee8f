// hub.cuh — the hub child lists' sorted warp list and the one-warp refresh
// of a hub's list (hub.cu has the design; step.cu refreshes per prompt).
#pragma once
#include "srt_internal.cuh"

namespace srt {
namespace {

__device__ unsigned long long g_refresh_stats[2];  // development: incremental, full-scan rebuilds

__device__ __forceinline__ unsigned long long child_key(uint32_t cnt, int32_t tok) {
  return ((unsigned long long)cnt << 32) | (0xFFFFFFFFu - (uint32_t)tok);  // larger = better
}

// A sorted (descending) warp list of up to 64 keys: lane i holds entries i and i + 32.
struct KeyList {
  unsigned long long k0, k1;
  uint32_t v0, v1;
  int size;
  __device__ __forceinline__ unsigned long long key_at(int j) const {
    return j < 32 ? __shfl_sync(0xffffffffu, k0, j) : __shfl_sync(0xffffffffu, k1, j - 32);
  }
  __device__ __forceinline__ void insert(unsigned long long k, uint32_t v, int lane, int K) {
    const int pos = __popc(__ballot_sync(0xffffffffu, lane < size && k0 > k)) +
                    __popc(__ballot_sync(0xffffffffu, lane + 32 < size && k1 > k));
    if (pos >= K) return;
    const unsigned long long uk0 = __shfl_up_sync(0xffffffffu, k0, 1);
    const uint32_t uv0 = __shfl_up_sync(0xffffffffu, v0, 1);
    const unsigned long long uk1 = __shfl_up_sync(0xffffffffu, k1, 1);
    const uint32_t uv1 = __shfl_up_sync(0xffffffffu, v1, 1);
    const unsigned long long lk = __shfl_sync(0xffffffffu, k0, 31);
    const uint32_t lv = __shfl_sync(0xffffffffu, v0, 31);
    if (lane + 32 >= pos) {
      if (lane + 32 == pos) { k1 = k; v1 = v; }
      else if (lane == 0) { k1 = lk; v1 = lv; }
      else { k1 = uk1; v1 = uv1; }
    }
    if (lane >= pos) {
      if (lane == pos) { k0 = k; v0 = v; }
      else { k0 = uk0; v0 = uv0; }
    }
    size = min(size + 1, K);
  }
  // offer 32 candidates (one per lane): the ones that beat the current last entry enter
  __device__ __forceinline__ void offer(bool valid, unsigned long long k, uint32_t v, int lane,
                                       int K) {
    const unsigned long long bar = size == K ? key_at(K - 1) : 0ull;
    unsigned pending = __ballot_sync(0xffffffffu, valid && (size < K || k > bar));
    while (pending) {
      const int src = __ffs(pending) - 1;
      pending &= pending - 1;
      const unsigned long long kk = __shfl_sync(0xffffffffu, k, src);
      const uint32_t vv = __shfl_sync(0xffffffffu, v, src);
      if (size == K && kk <= key_at(K - 1)) continue;
      insert(kk, vv, lane, K);
    }
  }
};

// One warp rebuilds hub u's list (prompt p's partition) if it is not valid:
// the previous list's last count bounds the threshold from below (counts
// only grow), else a lane-wise top-2 pass over the children picks one; then
// every child at or above it is ranked into a sorted warp list of K entries.
// Ordinary loads: the fused step orders them after the acquire of the
// prompt's release (step.cu).
// The caller orders it before any reader of p's lists.
constexpr int RANK_CAP = 192;  // candidates ranked in shared memory (else serial inserts)

// Write the top K of n candidates (ids cid[], keys key[] in shared memory,
// distinct nonzero keys) to list slot `slot` by rank, and its header.
__device__ __forceinline__ void write_ranked(const DevCache& c, uint32_t slot, uint32_t u,
                                             uint32_t nch, uint32_t csum, const uint32_t* cid,
                                             const unsigned long long* key, int n, int K,
                                             int lane) {
  const size_t e = (size_t)slot * HUB_K;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    const unsigned long long kj = j < n ? key[j] : 0ull;
    uint32_t rank = 0;
    for (int i = 0; i < n; ++i) rank += key[i] > kj;
    if (j < n && rank < (uint32_t)K) {
      c.hub_child[e + rank] = cid[j];
      c.hub_tok[e + rank] = (int32_t)(0xFFFFFFFFu - (uint32_t)kj);
      c.hub_cnt[e + rank] = (uint32_t)(kj >> 32);
    }
  }
  __syncwarp();
  if (lane == 0) {
    c.hub_len[slot] = (uint32_t)min(n, K);
    c.hub_nch[slot] = nch;
    c.hub_csum[slot] = csum;
    c.hub_node[slot] = u;
  }
  __syncwarp();
}

// sid: null, or >= RANK_CAP * 3 words of this warp's shared memory (the
// candidates at or above the threshold are then ranked in parallel there
// unless there are more than RANK_CAP of them)
__device__ void refresh_hub_warp(const DevCache& c, int32_t p, uint32_t u, int lane,
                                 uint32_t* sid = nullptr) {
  if (u >= c.H) return;  // roots are never expanded
  const uint4 r = *rec_of(c, u);
  const uint32_t nch = r.x;
  if (nch <= HUB_MIN) return;
  const uint32_t slot = hub_slot(c, p, u);
  const bool same = c.hub_node[slot] == u;
  if (same && c.hub_nch[slot] == nch && c.hub_csum[slot] == r.w) return;  // still valid
  const int K = min(HUB_K, c.Bmax);
  const uint32_t nb = blk_index(nch - 2) + 1;
  const uint32_t mybase = lane < (int)nb ? block_base(c, u, lane) : 0u;
  auto pos_of = [&](uint32_t k) {
    const uint32_t jj = k - 1;
    const uint32_t bi = blk_index(jj);
    const uint32_t base = __shfl_sync(0xffffffffu, mybase, (int)(bi & 31));
    return base + (jj - blk_start(bi));
  };
  constexpr int U4 = 8;  // child loads in flight per lane
  uint32_t thr = 0;
  if (same && c.hub_len[slot] == (uint32_t)K) {
    thr = c.hub_cnt[(size_t)slot * HUB_K + K - 1];
  } else {
    uint32_t t1 = 0, t2 = 0;
    for (uint32_t kb = 0; kb < nch; kb += U4 * 32) {
      uint32_t cv[U4];
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * 32 + lane;
        const uint32_t pos = pos_of(k >= 1 ? k : 1);  // (a shuffle: every lane)
        cv[q] = k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pos] : 0u;
      }
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        if (cv[q] > t1) { t2 = t1; t1 = cv[q]; }
        else if (cv[q] > t2) t2 = cv[q];
      }
    }
    for (int i = 0; i < K; ++i) {  // the K-th largest of the lanes' top-2 counts
      thr = __reduce_max_sync(0xffffffffu, t1);
      const unsigned who = __ballot_sync(0xffffffffu, t1 == thr);
      if (lane == __ffs(who) - 1) { t1 = t2; t2 = 0; }
    }
  }
  if (sid) {  // collect the candidates, then rank them
    uint32_t* cid = sid;
    unsigned long long* key = reinterpret_cast<unsigned long long*>(sid + RANK_CAP);
    int n = 0;
    bool over = false;
    for (uint32_t kb = 0; kb < nch && !over; kb += U4 * 32) {
      uint32_t cv[U4], pv[U4];
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * 32 + lane;
        pv[q] = pos_of(k >= 1 ? k : 1);
        cv[q] = k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pv[q]] : 0u;
      }
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * 32 + lane;
        const bool in = k < nch && cv[q] >= thr;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (!b) continue;
        if (n + __popc(b) > RANK_CAP) {
          over = true;
          break;
        }
        if (in) {
          const int at = n + __popc(b & lanemask_lt());
          uint32_t id;
          int32_t tk;
          if (k == 0) { id = r.y; tk = (int32_t)r.z; }
          else { id = c.slots[pv[q]]; tk = c.stok[pv[q]]; }
          cid[at] = id;
          key[at] = child_key(cv[q], tk);
        }
        n += __popc(b);
      }
    }
    __syncwarp();
    if (!over) {
      write_ranked(c, slot, u, nch, r.w, cid, key, n, K, lane);
      return;
    }
  }
  KeyList L{0ull, 0ull, NONE, NONE, 0};
  for (uint32_t kb = 0; kb < nch; kb += U4 * 32) {
    uint32_t cv[U4], pv[U4];
#pragma unroll
    for (int q = 0; q < U4; ++q) {
      const uint32_t k = kb + q * 32 + lane;
      pv[q] = pos_of(k >= 1 ? k : 1);
      cv[q] = k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pv[q]] : 0u;
    }
#pragma unroll
    for (int q = 0; q < U4; ++q) {
      const uint32_t k = kb + q * 32 + lane;
      const bool in = k < nch && cv[q] >= thr;
      if (__any_sync(0xffffffffu, in)) {
        uint32_t id = NONE;
        int32_t tk = 0;
        if (in) {
          if (k == 0) { id = r.y; tk = (int32_t)r.z; }
          else { id = c.slots[pv[q]]; tk = c.stok[pv[q]]; }
        }
        L.offer(in, child_key(cv[q], tk), id, lane, K);
      }
    }
  }
  const size_t e = (size_t)slot * HUB_K;
  if (lane < L.size) {
    c.hub_child[e + lane] = L.v0;
    c.hub_tok[e + lane] = (int32_t)(0xFFFFFFFFu - (uint32_t)L.k0);
    c.hub_cnt[e + lane] = (uint32_t)(L.k0 >> 32);
  }
  if (lane + 32 < L.size) {
    c.hub_child[e + lane + 32] = L.v1;
    c.hub_tok[e + lane + 32] = (int32_t)(0xFFFFFFFFu - (uint32_t)L.k1);
    c.hub_cnt[e + lane + 32] = (uint32_t)(L.k1 >> 32);
  }
  if (lane == 0) {
    c.hub_len[slot] = (uint32_t)L.size;
    c.hub_nch[slot] = nch;
    c.hub_csum[slot] = r.w;
    c.hub_node[slot] = u;
  }
  __syncwarp();
}

// Hub u's list rebuilt from its previous list and the children counted since
// it was built (kids[i * kstride], i < m, one count increment each): the new top K is
// among those (a child neither listed nor counted kept its count, below the
// old K-th entry's, which only grew).  Exact only when the touches account
// for the whole csum change since the build; otherwise (no previous list, a
// NONE touch = a hub a draft met without a list, lost touches) the full
// scan of refresh_hub_warp.  sid: >= RANK_CAP * 3 words (2.25 KB) of this warp's shared memory.
__device__ void refresh_hub_incr(const DevCache& c, int32_t p, uint32_t u, const uint32_t* kids,
                                 uint32_t m, uint32_t kstride, int lane, uint32_t* sid) {
  if (u >= c.H) return;
  const uint4 r = *rec_of(c, u);
  const uint32_t nch = r.x;
  if (nch <= HUB_MIN) return;
  const uint32_t slot = hub_slot(c, p, u);
  const bool same = c.hub_node[slot] == u;
  if (same && c.hub_nch[slot] == nch && c.hub_csum[slot] == r.w) return;  // still valid
  const int K = min(HUB_K, c.Bmax);
  bool incr = same && m <= 64 && c.hub_len[slot] == (uint32_t)K && r.w - c.hub_csum[slot] == m;
  const uint32_t k0 = lane < (int)m ? kids[(size_t)lane * kstride] : 0u;
  const uint32_t k1 = lane + 32 < (int)m ? kids[(size_t)(lane + 32) * kstride] : 0u;
  incr = incr && !__any_sync(0xffffffffu, k0 == NONE || k1 == NONE);
  if (lane == 0) atomicAdd(&g_refresh_stats[incr ? 0 : 1], 1ull);
  if (!incr) {
    refresh_hub_warp(c, p, u, lane, sid);
    return;
  }
  const size_t e = (size_t)slot * HUB_K;
  const int ncand = K + (int)m;  // <= 128
  if (lane < K) sid[lane] = c.hub_child[e + lane];
  if (lane + 32 < K) sid[lane + 32] = c.hub_child[e + lane + 32];
  if (lane < (int)m) sid[K + lane] = k0;
  if (lane + 32 < (int)m) sid[K + 32 + lane] = k1;
  __syncwarp();
  // every candidate's key (0 for a repeat of an earlier one), then its rank
  // among all of them: the entries of rank < K are the new list, written in
  // place -- no serial inserts (keys of distinct children are distinct: the
  // token breaks count ties)
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(sid + 128);
  unsigned long long key[4];
  uint32_t cid[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = q * 32 + lane;
    cid[q] = j < ncand ? sid[j] : NONE;
    bool keep = j < ncand;
    for (int i = 0; keep && i < j; ++i) keep = sid[i] != cid[q];  // first occurrence only
    key[q] = keep ? child_key(c.cnt[cid[q]], c.tok[cid[q]]) : 0ull;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q * 32 < ncand) skey[q * 32 + lane] = key[q];
  __syncwarp();
  uint32_t rank[4] = {0, 0, 0, 0};
  for (int i = 0; i < ncand; ++i) {
    const unsigned long long ki = skey[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) rank[q] += ki > key[q];
  }
  int nvalid = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    nvalid += __popc(__ballot_sync(0xffffffffu, key[q] != 0ull));
    if (key[q] != 0ull && rank[q] < (uint32_t)K) {
      c.hub_child[e + rank[q]] = cid[q];
      c.hub_tok[e + rank[q]] = (int32_t)(0xFFFFFFFFu - (uint32_t)key[q]);
      c.hub_cnt[e + rank[q]] = (uint32_t)(key[q] >> 32);
    }
  }
  __syncwarp();
  if (lane == 0) {
    c.hub_len[slot] = (uint32_t)min(nvalid, K);
    c.hub_nch[slot] = nch;
    c.hub_csum[slot] = r.w;
    c.hub_node[slot] = u;
  }
  __syncwarp();
}

}  // namespace
}  // namespace srt
