// insert.cu — srt_insert: batched, lock-free insertion of decoded and run-ahead
// spans into the per-prompt trees ("decoded outputs of running rollouts
// are inserted online into T_p and node counts are updated"; "index all
// substrings"; reading O1).
//
// Work decomposition: every window START i of every span is one work item
// (a thread); the thread walks the root along tokens[i .. min(i+D, to)-1],
// creating missing nodes (CAS on the edge hash) and adding 1 to the count of
// every node whose window ends at a new position (j >= from).  Items are
// flattened over spans by an exclusive scan so a 2k-token run-ahead span
// spreads over the whole grid instead of serialising in one warp.
// Roofline: latency-bound pointer chasing (<= D dependent hash probes per
// thread, each an L2/HBM round trip), reported as us per batch.
#include <cstdlib>

#include "srt_internal.cuh"
#include "accept.cuh"
#include "insert.cuh"

namespace srt {

namespace {

constexpr int PLAN_THREADS = 1024;  // one pass for the usual n <= 1024


// offs[s] = exclusive prefix sum of the window-start counts; offs[n] = total.
__global__ void __launch_bounds__(PLAN_THREADS)
k_insert_plan(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
              const int32_t* __restrict__ from, const int32_t* __restrict__ to,
              const int32_t* __restrict__ floor_, int32_t short_max, long long* __restrict__ offs) {
  __shared__ long long warp_tot[PLAN_THREADS / 32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t base = 0; base < n; base += PLAN_THREADS) {
    const int32_t s = base + threadIdx.x;
    long long w = 0;
    if (s < n) {
      const int32_t p = prompt_id[s];
      if (p < 0 || p >= c.P) {
        set_error(c, SRT_DEV_BAD_PROMPT);
      } else {
        const int32_t fl = floor_ ? floor_[s] : 0;
        const int32_t lo = span_lo(from[s], fl, c.D);
        const int32_t hi = to[s];
        if (hi > from[s] && hi > lo) w = hi - lo;
        // spans of <= short_max new positions go to the cursor kernel instead
        if (short_max >= 0 && hi - max(from[s], fl) <= short_max) w = 0;
      }
    }
    long long x = w;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      long long t = lane < PLAN_THREADS / 32 ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < PLAN_THREADS / 32) warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const long long before = carry + (wid ? warp_tot[wid - 1] : 0) + x - w;
    if (s < n) offs[s] = before;
    __syncthreads();
    if (threadIdx.x == PLAN_THREADS - 1) carry = before + w;
    __syncthreads();
  }
  if (threadIdx.x == 0) offs[n] = carry;
}


template <int NG>
__global__ void __launch_bounds__(CURSOR_WARPS * 32)
k_insert_cursor(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
                const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ from,
                const int32_t* __restrict__ to, const int32_t* __restrict__ floor_, int32_t short_max,
                uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  extern __shared__ __align__(16) unsigned char cur_smem[];
  const int w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * CURSOR_WARPS + w;
  if (s >= n) return;
  const int32_t p = prompt_id[s];
  if (p < 0 || p >= c.P) return;  // flagged by the plan kernel
  const CursorSmem S = carve_cursor_smem(cur_smem, w, c.D);
  cursor_insert_seq<NG>(c, S, s, p, from[s], to[s], seq_tok, stride, floor_, short_max, cursor, tag,
                        stats);
}

// D > 32: NG warps per sequence (one depth group each), one sequence per CTA.
template <int NG>
__global__ void __launch_bounds__(128)
k_insert_cursor_mw(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
                   const int32_t* __restrict__ seq_tok, int64_t stride,
                   const int32_t* __restrict__ from, const int32_t* __restrict__ to,
                   const int32_t* __restrict__ floor_, int32_t short_max,
                   uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  extern __shared__ __align__(16) unsigned char cur_smem[];
  const int32_t s = blockIdx.x;
  if (s >= n) return;
  const int32_t p = prompt_id[s];
  if (p < 0 || p >= c.P) return;  // flagged by the plan kernel
  CursorSmem S = carve_cursor_smem(cur_smem, threadIdx.x >> 5, c.D);
  S.A = carve_cursor_smem(cur_smem, 0, c.D).A;
  cursor_insert_seq<NG, true>(c, S, s, p, from[s], to[s], seq_tok, stride, floor_, short_max,
                              cursor, tag, stats);
}

template <int NG>
__global__ void __launch_bounds__(128)
k_accept_insert_mw(DevCache c, VerifyArgs a, const unsigned long long* __restrict__ result,
                   const int32_t* __restrict__ prompt_id, const int32_t* __restrict__ floor_,
                   uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  extern __shared__ __align__(16) unsigned char cur_smem[];
  __shared__ int32_t ctok[65];
  __shared__ int32_t acc[64];
  const int32_t s = blockIdx.x;
  if (s >= a.n) return;
  const int32_t t = a.seq_len[s];
  __syncthreads();
  if (threadIdx.x < 32) accept_seq(c, a, result, s, ctok, acc, threadIdx.x);
  __syncthreads();
  const int32_t t_end = a.seq_len[s];
  const int32_t p = prompt_id[s];
  if (p < 0 || p >= c.P) {
    if (threadIdx.x == 0) set_error(c, SRT_DEV_BAD_PROMPT);
    return;
  }
  CursorSmem S = carve_cursor_smem(cur_smem, threadIdx.x >> 5, c.D);
  S.A = carve_cursor_smem(cur_smem, 0, c.D).A;
  cursor_insert_seq<NG, true>(c, S, s, p, t, t_end, a.seq_tok, a.stride, floor_, INT_MAX, cursor,
                              tag, stats);
}

// Fused accept + cursor insert (srt_verify_insert_cursor): each warp commits
// its sequence (accept.cuh) and inserts the committed span through its cursor
// right away — no global round trip and no launch between the two stages.
// Every span goes through the cursor (a commit is at most Bmax + 1 tokens).
template <int NG>
__global__ void __launch_bounds__(CURSOR_WARPS * 32)
k_accept_insert(DevCache c, VerifyArgs a, const unsigned long long* __restrict__ result,
                const int32_t* __restrict__ prompt_id, const int32_t* __restrict__ floor_,
                uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  extern __shared__ __align__(16) unsigned char cur_smem[];
  __shared__ int32_t ctok[CURSOR_WARPS][65];
  __shared__ int32_t acc[CURSOR_WARPS][64];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * CURSOR_WARPS + w;
  if (s >= a.n) return;
  const int32_t t = accept_seq(c, a, result, s, ctok[w], acc[w], lane);
  __syncwarp();
  const int32_t t_end = a.seq_len[s];  // (written by lane 0 of this warp)
  const int32_t p = prompt_id[s];
  if (p < 0 || p >= c.P) {
    if (lane == 0) set_error(c, SRT_DEV_BAD_PROMPT);
    return;
  }
  const CursorSmem S = carve_cursor_smem(cur_smem, w, c.D);
  cursor_insert_seq<NG>(c, S, s, p, t, t_end, a.seq_tok, a.stride, floor_, INT_MAX, cursor, tag,
                        stats);
}

// Walk insertion (spans longer than D, run-ahead spans, no cursor): every
// window start is one lane's walk from the root along tokens[i .. i+D) (new
// nodes created, windows ending at a new position counted).  A warp's 32
// walks advance one hop per step with the convergent probe (probe_edges);
// linking new nodes and the mirror counts of pending ones are logged and
// batched per warp exactly as in the cursor kernel.  Window starts are
// flattened over the spans by an exclusive scan (k_insert_plan) so a
// 2k-token run-ahead span spreads over the whole grid.
__global__ void __launch_bounds__(CURSOR_WARPS * 32)
k_insert_walk(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
              const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ from,
              const int32_t* __restrict__ to, const int32_t* __restrict__ floor_,
              const long long* __restrict__ offs, srt_insert_stats* stats) {
  extern __shared__ __align__(16) unsigned char cur_smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  CursorSmem S;
  {
    unsigned char* b = cur_smem + (size_t)w * cursor_warp_bytes(c.D);
    b += ((size_t)(c.D + 1) * 4 + 15) & ~size_t(15);
    b += ((size_t)(c.D + 1) + 15) & ~size_t(15);
    S.A = nullptr;
    S.fresh = nullptr;
    S.log_h = reinterpret_cast<uint32_t*>(b);
    S.log_par = S.log_h + LOGCAP;
    S.log_tok = reinterpret_cast<int32_t*>(S.log_par + LOGCAP);
    S.pend = reinterpret_cast<uint32_t*>(S.log_tok + LOGCAP);
    S.nlog = reinterpret_cast<int*>(S.pend + LOGCAP);
    S.dbuf = reinterpret_cast<uint4*>(S.nlog + 4);
    S.pdl = nullptr;
  }
  if (lane == 0) S.nlog[0] = S.nlog[1] = S.nlog[2] = 0;
  __syncwarp();
  const long long total = offs[n];
  unsigned windows = 0, incs = 0, created = 0;
  const long long stride_w = (long long)gridDim.x * CURSOR_WARPS * 32;
  for (long long base = ((long long)blockIdx.x * CURSOR_WARPS + w) * 32; base < total;
       base += stride_w) {
    const long long idx = base + lane;
    int32_t i = 0, j = 0, end = 0, f = 0, pr = 0;
    uint32_t u = NONE;
    const int32_t* toks = nullptr;
    if (idx < total) {
      int32_t lo_s = 0, hi_s = n - 1;  // span s: offs[s] <= idx < offs[s+1]
      while (lo_s < hi_s) {
        const int32_t mid = (lo_s + hi_s + 1) >> 1;
        if (offs[mid] <= idx) lo_s = mid; else hi_s = mid - 1;
      }
      const int32_t s = lo_s;
      f = from[s];
      i = span_lo(f, floor_ ? floor_[s] : 0, c.D) + (int32_t)(idx - offs[s]);
      toks = seq_tok + (int64_t)s * stride;
      pr = prompt_id[s];
      u = root_id(c, pr);
      end = min(i + c.D, to[s]);
      j = i;
      ++windows;
    }
    bool live = idx < total && j < end;
    int32_t tk_nx = live ? toks[j] : 0;
    while (__any_sync(0xffffffffu, live)) {
      int32_t tk = tk_nx;
      if (live) {
        tk_nx = j + 1 < end ? toks[j + 1] : 0;  // next hop's token, in flight during the probe
        if (tk < 0 || tk >= c.V) {
          set_error(c, SRT_DEV_OOV);
          live = false;
        }
      }
      const unsigned long long key[1] = {live ? edge_key(u, (uint32_t)tk) : 0ull};
      bool act[1] = {live};
      uint32_t hnew[1], aux[1];
      bool cre[1];
      probe_edges<1>(c, key, act, hnew, cre, aux);
      const bool a = act[0];
      const uint32_t h = hnew[0];
      const bool counted = a && j >= f;  // a window ends at a new position
      if (a) {
        if (cre[0]) c.tok[h] = tk;
        if (counted) {
          atomicAdd(&c.cnt[h], 1u);
          atomicAdd(&rec_of(c, u)->w, 1u);
          ++incs;
          if (!cre[0] && is_slot_word(aux[0])) atomicAdd(&c.scnt[aux[0]], 1u);
        }
      }
      dirty_push(c, S, counted && j - i >= 1 && j - i <= HUB_DIRTY_DEPTH, u, pr, h, lane);
      const unsigned mc = __ballot_sync(0xffffffffu, a && cre[0]);
      const unsigned mp = __ballot_sync(0xffffffffu, counted && !cre[0] && aux[0] == NONE);
      if (mc | mp) {
        int bc = 0, bp = 0;
        if (lane == 0) {
          bc = S.nlog[0];
          bp = S.nlog[1];
          S.nlog[0] = bc + __popc(mc);
          S.nlog[1] = bp + __popc(mp);
        }
        bc = __shfl_sync(0xffffffffu, bc, 0);
        bp = __shfl_sync(0xffffffffu, bp, 0);
        const unsigned lt = lanemask_lt();
        if (mc >> lane & 1) {
          const int e = bc + __popc(mc & lt);
          S.log_h[e] = h;
          S.log_par[e] = u;
          S.log_tok[e] = counted ? tk : (int32_t)((uint32_t)tk | 0x80000000u);
          ++created;
        }
        if (mp >> lane & 1) S.pend[bp + __popc(mp & lt)] = h;
      }
      __syncwarp();
      if (a) {
        u = h;
        ++j;
      }
      live = a && j < end;
      if (S.nlog[0] > LOGCAP - 32 || S.nlog[1] > LOGCAP - 32) cursor_flush(c, S, lane);
    }
  }
  cursor_flush(c, S, lane);
  dirty_flush(c, S, lane);
  count_created(c, created);
  if (stats) {
    unsigned long long a = windows, b = incs, d = created;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if (lane == 0 && (a | b | d)) {
      atomicAdd(&stats->windows, a);
      atomicAdd(&stats->increments, b);
      atomicAdd(&stats->nodes_created, d);
    }
  }
}

// One dump record per thread (srt_cache_load): the child of its parent (the
// previous level's node par_idx) labelled tok is created if missing and its
// count, mirror count and the parent's csum grow by the record's count.
__global__ void __launch_bounds__(256)
k_load_level(DevCache c, const uint32_t* __restrict__ parent_ids, const int32_t* __restrict__ par_idx,
             const int32_t* __restrict__ tok, const unsigned long long* __restrict__ cnt, int32_t n,
             uint32_t* __restrict__ out_ids) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned created = 0;
  if (i < n) {
    const uint32_t u = parent_ids[par_idx[i]];
    const int32_t tk = tok[i];
    uint32_t id = BAD;
    if (tk < 0 || tk >= c.V) {
      set_error(c, SRT_DEV_OOV);
    } else if (u < BAD) {
      uint32_t pos;
      id = get_or_create(c, u, tk, &pos, created);
      if (id < BAD) {
        const uint32_t k = (uint32_t)cnt[i];
        atomicAdd(&c.cnt[id], k);
        if (is_slot_word(pos)) atomicAdd(&c.scnt[pos], k);
        atomicAdd(&rec_of(c, u)->w, k);
      }
    }
    out_ids[i] = id;
  }
  count_created(c, created);
}

}  // namespace

cudaError_t launch_load_level(const DevCache& c, const uint32_t* parent_ids, const int32_t* par_idx,
                              const int32_t* tok, const unsigned long long* cnt, int32_t n,
                              uint32_t* out_ids, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  k_load_level<<<(n + 255) / 256, 256, 0, stream>>>(c, parent_ids, par_idx, tok, cnt, n, out_ids);
  return cudaGetLastError();
}

cudaError_t set_insert_profile(long long* buf) {
  return cudaMemcpyToSymbol(g_ins_prof, &buf, sizeof(buf));
}

cudaError_t launch_insert_plan(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* from, const int32_t* to, const int32_t* floor_,
                               int32_t short_max, long long* scratch, cudaStream_t stream) {
  carveout_once<k_insert_plan>();
  k_insert_plan<<<1, PLAN_THREADS, 0, stream>>>(c, n, prompt_id, from, to, floor_, short_max,
                                                scratch);
  return cudaGetLastError();
}

cudaError_t launch_insert_walk(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* seq_tok, int64_t stride, const int32_t* from,
                               const int32_t* to, const int32_t* floor_, srt_insert_stats* stats,
                               const long long* scratch, cudaStream_t stream) {
  const size_t smem = insert_cursor_smem(c.D);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_insert_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_insert_walk<<<num_sms() * 4, CURSOR_WARPS * 32, smem, stream>>>(c, n, prompt_id, seq_tok, stride,
                                                                    from, to, floor_, scratch, stats);
  return cudaGetLastError();
}

size_t insert_cursor_smem(int32_t D) { return (size_t)CURSOR_WARPS * cursor_warp_bytes(D); }

cudaError_t launch_accept_insert(const DevCache& c, const VerifyArgs& a,
                                 const unsigned long long* result, const int32_t* prompt_id,
                                 const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                                 srt_insert_stats* stats, cudaStream_t stream) {
  const int ng = (c.D + 31) >> 5;
  if (ng >= 2) {  // one sequence per CTA, one warp per depth group
    const size_t smem = (size_t)ng * cursor_warp_bytes(c.D);
    auto kern = ng == 2 ? k_accept_insert_mw<2> : ng == 3 ? k_accept_insert_mw<3>
                                                          : k_accept_insert_mw<4>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<a.n, ng * 32, smem, stream>>>(c, a, result, prompt_id, floor_, cursor, tag, stats);
    return cudaGetLastError();
  }
  const size_t smem = insert_cursor_smem(c.D);
  auto kern = k_accept_insert<1>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<(a.n + CURSOR_WARPS - 1) / CURSOR_WARPS, CURSOR_WARPS * 32, smem, stream>>>(
      c, a, result, prompt_id, floor_, cursor, tag, stats);
  return cudaGetLastError();
}

cudaError_t launch_insert_cursor(const DevCache& c, int32_t n, const int32_t* prompt_id,
                                 const int32_t* seq_tok, int64_t stride, const int32_t* from,
                                 const int32_t* to, const int32_t* floor_, int32_t short_max,
                                 uint32_t* cursor, uint32_t tag, srt_insert_stats* stats,
                                 cudaStream_t stream) {
  const int ng = (c.D + 31) >> 5;
  if (ng >= 2) {  // one sequence per CTA, one warp per depth group
    const size_t smem = (size_t)ng * cursor_warp_bytes(c.D);
    auto kern = ng == 2 ? k_insert_cursor_mw<2> : ng == 3 ? k_insert_cursor_mw<3>
                                                          : k_insert_cursor_mw<4>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<n, ng * 32, smem, stream>>>(c, n, prompt_id, seq_tok, stride, from, to, floor_,
                                       short_max, cursor, tag, stats);
    return cudaGetLastError();
  }
  const size_t smem = insert_cursor_smem(c.D);
  auto kern = k_insert_cursor<1>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<(n + CURSOR_WARPS - 1) / CURSOR_WARPS, CURSOR_WARPS * 32, smem, stream>>>(
      c, n, prompt_id, seq_tok, stride, from, to, floor_, short_max, cursor, tag, stats);
  return cudaGetLastError();
}

}  // namespace srt
