// hub.cu — the hub child lists: for every node with more than
// HUB_MIN children that an insert touched, its top HUB_K children by (count
// desc, token asc), so that srt_draft expands a hub in O(cap) instead of
// ranking thousands of children at every pop.  Siblings rank by count (score
// is strictly monotone in it, O6) with ties by token (O8), so the first cap
// entries of the list are exactly the children that can enter a frontier of
// cap entries.  A list is used only while its node's child count and csum are
// unchanged (counts only grow), so it is never stale.
//
// After every insert call: the inserts logged the shallow parents whose csum
// they changed and srt_draft logged the hubs it had to expand without a valid
// list (the dirty list); k_hub_pick elects one refresher per cache
// slot (a node listed several times, or two hubs sharing a slot, refresh
// once), and k_hub_refresh rebuilds each elected list with one CTA: a count
// threshold first (lane-wise top-2 counts), then every warp keeps a sorted
// top-K of its share of the children at or above it, the lists are merged by rank.
#include "srt_internal.cuh"
#include "hub.cuh"

namespace srt {

namespace {

constexpr int REFRESH_WARPS = 8;

// Each dirty hub whose list is stale claims its cache slot for this refresh
// generation with one CAS: the first claim of a slot wins (a node listed
// several times refreshes once; of two hubs sharing a slot one refreshes, the
// other keeps the full scan until a later refresh) and joins the work list.
__global__ void k_hub_pick(DevCache c, uint2* work, uint32_t* work_n) {
  const uint32_t call = c.dirty_n[1] + 1;  // this refresh's generation
  const uint32_t n = min(*c.dirty_n, DIRTY_CAP);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 du = c.dirty[i];
    const uint32_t u = du.x;
    if (u >= c.H || du.y >= (uint32_t)c.P) continue;  // roots are never expanded
    const uint4 r = *rec_of(c, u);
    if (r.x <= HUB_MIN) continue;
    const uint32_t slot = hub_slot(c, (int32_t)du.y, u);
    // (a list that is still valid needs no rebuild)
    if (c.hub_node[slot] == u && c.hub_nch[slot] == r.x && c.hub_csum[slot] == r.w) continue;
    const unsigned long long c0 = c.hub_claim[slot];
    if ((uint32_t)(c0 >> 32) == call) continue;  // claimed in this generation already
    if (atomicCAS(&c.hub_claim[slot], c0, ((unsigned long long)call << 32) | u) != c0) continue;
    work[atomicAdd(work_n, 1u)] = du;
  }
}

__global__ void __launch_bounds__(REFRESH_WARPS * 32)
k_hub_refresh(DevCache c, const uint2* __restrict__ work, const uint32_t* work_n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.dirty_n[1] += 1;  // next refresh's generation
    c.dirty_n[0] = 0;   // k_hub_pick consumed the list
  }
  __shared__ unsigned long long sk[REFRESH_WARPS][HUB_K];
  __shared__ uint32_t sv[REFRESH_WARPS][HUB_K];
  __shared__ int sn[REFRESH_WARPS];
  __shared__ uint32_t sthr[REFRESH_WARPS];
  constexpr int WCAP = 128;  // a warp's candidates ranked in shared memory (else serial inserts)
  __shared__ unsigned long long ck[REFRESH_WARPS][WCAP];
  __shared__ uint32_t cv_id[REFRESH_WARPS][WCAP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int K = min(HUB_K, c.Bmax);  // the draft never needs more than Bmax of them
  const uint32_t nw = *work_n;
  for (uint32_t it = blockIdx.x; it < nw; it += gridDim.x) {
    const uint2 wu = work[it];
    const uint32_t u = wu.x;
    const uint4 r = *rec_of(c, u);
    const uint32_t nch = r.x;
    const uint32_t nb = blk_index(nch - 2) + 1;
    const uint32_t mybase = lane < (int)nb ? block_base(c, u, lane) : 0u;
    constexpr int U4 = 4;  // slices in flight per warp
    constexpr uint32_t STEP = REFRESH_WARPS * 32;
    // child k (0 = the inline first child) -> its count; its id and token are
    // loaded only for the few children at or above the threshold
    auto pos_of = [&](uint32_t k) {
      const uint32_t jj = k - 1;
      const uint32_t bi = blk_index(jj);
      const uint32_t base = __shfl_sync(0xffffffffu, mybase, (int)(bi & 31));
      return base + (jj - blk_start(bi));
    };
    auto load_cnt = [&](uint32_t k) -> uint32_t {
      const uint32_t pos = pos_of(k >= 1 ? k : 1);
      return k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pos] : 0u;
    };
    // The previous list of this node (if any) bounds the threshold from below:
    // counts only grow, so its K children still have counts >= its last
    // entry's, and no child below that count can enter the new list.
    const uint32_t slot = hub_slot(c, (int32_t)wu.y, u);
    uint32_t thr = 0;
    if (c.hub_node[slot] == u && c.hub_len[slot] == (uint32_t)K) {
      thr = c.hub_cnt[(size_t)slot * HUB_K + K - 1];
    } else {
      // pass 1: every lane keeps the two largest counts of its children; a warp's
      // K-th largest of those 64 has >= K children at or above it, so children
      // below the largest such threshold over the warps can never be in the list
      uint32_t t1 = 0, t2 = 0;
      for (uint32_t kb = (uint32_t)w * 32; kb < nch; kb += U4 * STEP) {
        uint32_t cv[U4];
#pragma unroll
        for (int q = 0; q < U4; ++q) cv[q] = load_cnt(kb + q * STEP + lane);
#pragma unroll
        for (int q = 0; q < U4; ++q) {
          const uint32_t cn = cv[q];
          if (cn > t1) { t2 = t1; t1 = cn; }
          else if (cn > t2) t2 = cn;
        }
      }
      for (int i = 0; i < K; ++i) {
        thr = __reduce_max_sync(0xffffffffu, t1);
        const unsigned who = __ballot_sync(0xffffffffu, t1 == thr);
        if (lane == __ffs(who) - 1) { t1 = t2; t2 = 0; }
      }
      if (lane == 0) sthr[w] = thr;
      __syncthreads();
      thr = 0;
      for (int o = 0; o < REFRESH_WARPS; ++o) thr = max(thr, sthr[o]);
    }
    // pass 2: rank only the children at or above the threshold: each warp
    // collects its slice's candidates and sorts them by rank (in parallel,
    // from shared memory) into its top-K list, unless it has more than WCAP
    // of them (then serial inserts into a sorted warp list)
    int n = 0;
    bool over = false;
    for (uint32_t kb = (uint32_t)w * 32; kb < nch && !over; kb += U4 * STEP) {
      uint32_t cv[U4], pv[U4];
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * STEP + lane;
        pv[q] = pos_of(k >= 1 ? k : 1);
        cv[q] = k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pv[q]] : 0u;
      }
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * STEP + lane;
        const bool in = k < nch && cv[q] >= thr;
        const unsigned b = __ballot_sync(0xffffffffu, in);
        if (!b) continue;
        if (n + __popc(b) > WCAP) {
          over = true;
          break;
        }
        if (in) {
          const int at = n + __popc(b & lanemask_lt());
          uint32_t id;
          int32_t tk;
          if (k == 0) { id = r.y; tk = (int32_t)r.z; }
          else { id = c.slots[pv[q]]; tk = c.stok[pv[q]]; }
          cv_id[w][at] = id;
          ck[w][at] = child_key(cv[q], tk);
        }
        n += __popc(b);
      }
    }
    __syncwarp();
    if (!over) {
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        const unsigned long long kj = j < n ? ck[w][j] : 0ull;
        int rank = 0;
        for (int i = 0; i < n; ++i) rank += ck[w][i] > kj;
        if (j < n && rank < K) {
          sk[w][rank] = kj;
          sv[w][rank] = cv_id[w][j];
        }
      }
      if (lane == 0) sn[w] = min(n, K);
    }
    KeyList L{0ull, 0ull, NONE, NONE, 0};
    for (uint32_t kb = (uint32_t)w * 32; over && kb < nch; kb += U4 * STEP) {
      uint32_t cv[U4], pv[U4];
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * STEP + lane;
        pv[q] = pos_of(k >= 1 ? k : 1);
        cv[q] = k == 0 ? c.cnt[r.y] : k < nch ? c.scnt[pv[q]] : 0u;
      }
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const uint32_t k = kb + q * STEP + lane;
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
    if (over) {
      sk[w][lane] = L.k0;
      sv[w][lane] = L.v0;
      sk[w][lane + 32] = L.k1;
      sv[w][lane + 32] = L.v1;
      if (lane == 0) sn[w] = L.size;
    }
    __syncthreads();
    // Merge the warps' sorted lists in parallel: an entry's place in the union
    // is its index in its own list plus the number of larger keys in each of
    // the others (binary searches in shared memory; keys are unique: one
    // child each), and the entries that place below K are written there.
    const size_t e = (size_t)slot * HUB_K;
    for (int i = lane; i < sn[w]; i += 32) {
      const unsigned long long kk = sk[w][i];
      int rank = i;
      for (int o = 0; o < REFRESH_WARPS; ++o) {
        if (o == w) continue;
        int lo = 0, hi = sn[o];
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (sk[o][mid] > kk) lo = mid + 1; else hi = mid;
        }
        rank += lo;
      }
      if (rank < K) {
        c.hub_child[e + rank] = sv[w][i];
        c.hub_tok[e + rank] = (int32_t)(0xFFFFFFFFu - (uint32_t)kk);
        c.hub_cnt[e + rank] = (uint32_t)(kk >> 32);
      }
    }
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int o = 0; o < REFRESH_WARPS; ++o) tot += sn[o];
      c.hub_len[slot] = (uint32_t)min(tot, K);
      c.hub_nch[slot] = nch;
      c.hub_csum[slot] = r.w;
      c.hub_node[slot] = u;  // (read by later kernels only)
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_hub_refresh(const DevCache& c, uint32_t call, uint32_t* work, uint32_t* work_n,
                               cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(work_n, 0, 4, stream);
  if (e != cudaSuccess) return e;
  const int g = num_sms() * 4;
  (void)call;
  k_hub_pick<<<g, 256, 0, stream>>>(c, reinterpret_cast<uint2*>(work), work_n);
  k_hub_refresh<<<num_sms() * 8, REFRESH_WARPS * 32, 0, stream>>>(
      c, reinterpret_cast<const uint2*>(work), work_n);
  return cudaGetLastError();
}

}  // namespace srt
