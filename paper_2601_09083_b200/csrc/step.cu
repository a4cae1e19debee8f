// step.cu — the fused tree step after the forward pass: the
// commit of step k (first-mismatch walk), the insertion of the
// committed spans into the trees ("inserted online"), the hub-list
// refresh and the draft of step k + 1 in ONE persistent launch,
// ordered per prompt instead of by kernel boundaries.
//
// Reading O14 only orders draft(k + 1) after every insert <= k of the SAME
// tree: prompts are independent (trees share no node), so prompt p's drafts
// may start as soon as p's own sequences are committed and inserted and p's
// hub lists are rebuilt, while other prompts are still inserting.  The
// separate kernels pay max(insert) + max(refresh) + max(draft) per step (each
// launch waits for its slowest warp: the longest accepted span, the biggest
// hub, the deepest expansion); here a step pays roughly the max over prompts
// of insert_p + refresh_p + draft_p.
//
// One warp per sequence (D <= 32), all CTAs resident (the grid is sized by
// the occupancy calculator), two phases per warp:
//  1. accept + cursor insert of its sequences (accept.cuh, insert.cuh); the
//     warp that completes a prompt's count rebuilds that prompt's dirty hub
//     lists (hub.cuh, one warp; prompt-partitioned slots, so no other
//     prompt's draft reads them) and then releases the prompt;
//  2. the draft of its sequences (draft.cuh), each after its prompt's
//     release; the warp completing the last draft writes the row offsets.
// Phase 1 never waits on phase 2, and every warp finishes its phase-1 work
// before it waits, so the waits always end.  Outputs are exactly those of
// srt_verify_insert_cursor followed by srt_draft_cursor (the hub lists only
// change how fast a draft is found, never which).
#define SRT_COHERENT_LOADS 1  // tree data written by other warps of this launch
#include "srt_internal.cuh"
#include "accept.cuh"
#include "insert.cuh"
#include "draft.cuh"
#include "hub.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace srt {

namespace {

constexpr int STEP_WARPS = 4;

struct StepDraftArgs {
  const int32_t* pos_base;  // nullable (read after the commit: may alias seq_len)
  int32_t* match_len;
  int32_t* draft_len;
  int32_t* draft_tok;
  int32_t* draft_parent;
  int32_t* draft_depth;
  int32_t* draft_pos;
  uint64_t* draft_mask;
  int64_t* row_offsets;
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// per prompt: sequences in this batch (pcount), and the counters cleared
__global__ void __launch_bounds__(1024) k_step_prep(DevCache c, int32_t n,
                                                    const int32_t* __restrict__ prompt_id) {
  for (int32_t i = threadIdx.x; i < c.P; i += blockDim.x) {
    c.st_pcount[i] = 0;
    c.st_pdone[i] = 0;
    c.st_pready[i] = 0;
    c.st_pnd[i] = 0;
    c.st_pnext[i] = 0;
    c.st_pfin[i] = 0;
  }
  if (threadIdx.x == 0) *c.st_ndone = 0;
  __syncthreads();
  for (int32_t s = threadIdx.x; s < n; s += blockDim.x) {
    const int32_t p = prompt_id[s];
    if (p >= 0 && p < c.P) atomicAdd(&c.st_pcount[p], 1u);
  }
}

// row_offsets[s] = sum_{s' < s} (draft_len[s'] + 1), one warp
__device__ void row_offsets_warp(int32_t n, const int32_t* draft_len, int64_t* row_offsets,
                                 int lane) {
  long long carry = 0;
  for (int32_t b = 0; b < n; b += 32) {
    const int32_t s = b + lane;
    const long long w = s < n ? (long long)ld_acquire_u32((const uint32_t*)&draft_len[s]) + 1 : 0;
    long long x = w;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (s < n) row_offsets[s] = carry + x - w;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) row_offsets[n] = carry;
}

// development profile: per warp {start, phase-1 end, release seen, end,
// refresh cycles, hubs refreshed, sequences, 0} (globaltimer ns / cycles)
__device__ unsigned long long* g_step_prof = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__host__ __device__ __forceinline__ size_t tree_step_smem_per_warp_dev(int32_t D) {
  const size_t per_warp = (cursor_warp_bytes(D) + 2 * 65 * 4 + 15) & ~size_t(15);
  const size_t dr = 64 * 8 + 64 * sizeof(Ent);
  return per_warp > dr ? per_warp : dr;
}

// Sort prompt p's n touch pairs (hub, child) by hub in shared memory (sk:
// >= 256 u64 of this warp's) and write them back with the refresh tasks:
// task t = the pairs [lo, hi) of one hub that needs a list (more than HUB_MIN
// children, no valid list) -- the other touched parents are dropped here, one
// record load per distinct parent, all lanes at once.  Returns the task count.
__device__ uint32_t group_touches(const DevCache& c, int32_t p, uint32_t* pdl, uint32_t n,
                                  unsigned long long* sk, int lane) {
  uint2* const task = reinterpret_cast<uint2*>(pdl + 2 + 2 * PDIRTY_CAP);
  for (uint32_t i = lane; i < n; i += 32)
    sk[i] = ((unsigned long long)pdl[2 + 2 * i] << 32) | pdl[3 + 2 * i];
  __syncwarp();
  constexpr int PER = (PDIRTY_CAP + 31) / 32;
  unsigned long long key[PER];
  uint32_t rank[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const uint32_t i = lane + 32 * k;
    key[k] = i < n ? sk[i] : ~0ull;
    rank[k] = 0;
  }
  const int per = (int)((n + 31) / 32);  // (warp-uniform) key slots in use
  for (uint32_t j = 0; j < n; ++j) {  // rank = smaller keys + equal keys before it
    const unsigned long long kj = sk[j];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (k >= per) break;
      const uint32_t i = lane + 32 * k;
      rank[k] += kj < key[k] || (kj == key[k] && j < i);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (lane + 32 * k < n) sk[rank[k]] = key[k];
  __syncwarp();
  uint32_t nt = 0;
  for (uint32_t b = 0; b < n; b += 32) {
    const uint32_t i = b + lane;
    const bool in = i < n;
    uint32_t u = NONE;
    if (in) {
      u = (uint32_t)(sk[i] >> 32);
      pdl[2 + 2 * i] = u;
      pdl[3 + 2 * i] = (uint32_t)sk[i];
    }
    bool first = in && (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32));
    if (first) {  // a parent that needs a (new) list?
      first = false;
      if (u < c.H) {
        const uint4 r = *rec_of(c, u);
        if (r.x > HUB_MIN) {
          const uint32_t slot = hub_slot(c, p, u);
          first = !(c.hub_node[slot] == u && c.hub_nch[slot] == r.x && c.hub_csum[slot] == r.w);
        }
      }
    }
    uint32_t hi = i + 1;  // the hub's pairs end where the next hub's begin
    while (first && hi < n && (sk[hi] >> 32) == u) ++hi;
    const unsigned fm = __ballot_sync(0xffffffffu, first);
    if (first) task[nt + __popc(fm & lanemask_lt())] = make_uint2(i, hi);
    nt += __popc(fm);
  }
  __syncwarp();
  return nt;
}

// Claim and run prompt p's hub refresh tasks until none is left; the warp
// finishing the last one resets p's touch list and marks p ready (2).
// Returns the cycles spent; hubs counts the tasks run.
__device__ long long refresh_tasks(const DevCache& c, int32_t p, int lane,
                                   unsigned long long& hubs, uint32_t* sid,
                                   bool* finisher = nullptr) {
  const long long t0 = clock64();
  uint32_t* const pdl = c.pdirty + (size_t)p * PDIRTY_WORDS;
  const uint2* const task = reinterpret_cast<const uint2*>(pdl + 2 + 2 * PDIRTY_CAP);
  const uint32_t nd = c.st_pnd[p];
  while (true) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(&c.st_pnext[p], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nd) break;
    const uint2 t = task[i];
    refresh_hub_incr(c, p, pdl[2 + 2 * t.x], pdl + 3 + 2 * t.x, t.y - t.x, 2, lane, sid);
    ++hubs;
    __syncwarp();
    uint32_t fin = 0;
    if (lane == 0) {
      __threadfence();  // this list before the count
      fin = atomicAdd(&c.st_pfin[p], 1u) + 1 == nd;
    }
    if (__shfl_sync(0xffffffffu, fin, 0)) {
      if (lane == 0) {
        pdl[0] = 0;  // consumed (this prompt's drafts log into it again)
        __threadfence();
        atomicExch(&c.st_pready[p], 2u);  // release prompt p to its drafts
      }
      __syncwarp();
      if (finisher) *finisher = true;
      break;
    }
  }
  return clock64() - t0;
}

// NG = 1 (D <= 32): 4 warps per CTA, one warp per sequence in both phases.
// NG > 1 (D <= 32 NG): NG warps per CTA; phase 1 inserts one sequence per CTA
// (one warp per depth group, insert.cuh's multi-warp cursor insert), phase
// 2 drafts one sequence per warp as before.
template <int NG, int WPC_ = (NG == 1 ? STEP_WARPS : NG)>
__global__ void __launch_bounds__(WPC_ * 32)
k_tree_step(DevCache c, VerifyArgs a, const unsigned long long* __restrict__ result,
            const int32_t* __restrict__ prompt_id, const int32_t* __restrict__ floor_,
            uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats,
            StepDraftArgs d) {
  constexpr int WPC = WPC_;  // warps per CTA
  extern __shared__ __align__(16) unsigned char step_smem[];
  __shared__ uint32_t sh_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t cw = cursor_warp_bytes(c.D);
  const size_t per_warp = (cw + 2 * 65 * 4 + 15) & ~size_t(15);
  unsigned char* mine = step_smem + (size_t)w * (per_warp > 64 * 8 + 64 * sizeof(Ent)
                                                     ? per_warp
                                                     : 64 * 8 + 64 * sizeof(Ent));
  const int32_t gw = blockIdx.x * WPC + w;
  const int32_t W = gridDim.x * WPC;
  const int32_t n = a.n;
  unsigned long long* const prof = g_step_prof;
  unsigned long long pf[8] = {prof ? gtime() : 0ull, 0, 0, 0, 0, 0, 0, 0};

  // ---- phase 1: commit + insert; the last of a prompt rebuilds its hub lists
  // (the warp that completes a prompt's count groups its touches and
  // publishes them as refresh tasks; it and the prompt's waiting draft warps
  // share the tasks)
  auto publish_tasks = [&](int32_t p, uint32_t* pdl) {
    __threadfence();  // every sibling's updates (they fenced before counting)
    const uint32_t n_t = min(*(volatile uint32_t*)pdl, PDIRTY_CAP);
    const uint32_t nd = group_touches(c, p, pdl, n_t,
                                      reinterpret_cast<unsigned long long*>(mine), lane);
    if (lane == 0) {
      c.st_pnd[p] = nd;
      if (!nd) pdl[0] = 0;
      __threadfence();
      atomicExch(&c.st_pready[p], nd ? 1u : 2u);
    }
    __syncwarp();
  };
  if (NG == 1) {
    CursorSmem S = carve_cursor_smem(mine, 0, c.D);
    int32_t* ctok = reinterpret_cast<int32_t*>(mine + cw);
    int32_t* acc = ctok + 65;
    for (int32_t s = gw; s < n; s += W) {
      const int32_t t = accept_seq(c, a, result, s, ctok, acc, lane);
      __syncwarp();
      const int32_t t_end = a.seq_len[s];  // (written by lane 0 of this warp)
      const int32_t p = prompt_id[s];
      if (p < 0 || p >= c.P) {
        if (lane == 0) set_error(c, SRT_DEV_BAD_PROMPT);
        continue;
      }
      uint32_t* const pdl = c.pdirty + (size_t)p * PDIRTY_WORDS;
      S.pdl = pdl;
      cursor_insert_seq<1>(c, S, s, p, t, t_end, a.seq_tok, a.stride, floor_, INT_MAX, cursor, tag,
                           stats);
      __syncwarp();
      uint32_t last = 0;
      if (lane == 0) {
        __threadfence();  // this sequence's tree updates before the prompt's count
        last = atomicAdd(&c.st_pdone[p], 1u) + 1 == c.st_pcount[p];
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        publish_tasks(p, pdl);
        pf[4] += refresh_tasks(c, p, lane, pf[5], reinterpret_cast<uint32_t*>(mine));
      }
    }
  } else {
    // one sequence per CTA: warp 0 commits it, every warp inserts its depth
    // group (S.A shared: warp 0's slice), warp 0 counts it toward the prompt
    CursorSmem S = carve_cursor_smem(step_smem, 0, c.D);  // (stride set below)
    for (int32_t s = blockIdx.x; s < n; s += gridDim.x) {
      const int32_t t = a.seq_len[s];
      __syncthreads();
      if (w == 0) {
        int32_t* ctok = reinterpret_cast<int32_t*>(mine + cw);
        accept_seq(c, a, result, s, ctok, ctok + 65, lane);
      }
      __syncthreads();
      const int32_t t_end = a.seq_len[s];
      const int32_t p = prompt_id[s];
      if (p < 0 || p >= c.P) {
        if (threadIdx.x == 0) set_error(c, SRT_DEV_BAD_PROMPT);
        continue;
      }
      uint32_t* const pdl = c.pdirty + (size_t)p * PDIRTY_WORDS;
      S = carve_cursor_smem(mine, 0, c.D);
      S.A = carve_cursor_smem(step_smem, 0, c.D).A;
      S.pdl = pdl;
      cursor_insert_seq<NG, true>(c, S, s, p, t, t_end, a.seq_tok, a.stride, floor_, INT_MAX,
                                  cursor, tag, stats);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        sh_last = atomicAdd(&c.st_pdone[p], 1u) + 1 == c.st_pcount[p];
      }
      __syncthreads();
      if (sh_last) {
        if (w == 0) publish_tasks(p, pdl);
        __syncthreads();
        pf[4] += refresh_tasks(c, p, lane, pf[5], reinterpret_cast<uint32_t*>(mine));
      }
      __syncthreads();
    }
  }
  __syncwarp();
  if (prof) pf[1] = gtime();
  // ---- phase 2: the next drafts, each once its prompt is released
  {
    unsigned long long* M = reinterpret_cast<unsigned long long*>(mine);
    Ent* merge = reinterpret_cast<Ent*>(mine + 64 * 8);
    for (int32_t s = gw; s < n; s += W) {
      const int32_t p = prompt_id[s];
      if (p >= 0 && p < c.P) {
        // wait for the prompt's inserts, help with its hub refresh tasks, wait
        // for the last of them
        while (true) {
          uint32_t stt = 0;
          if (lane == 0) stt = ld_acquire_u32(&c.st_pready[p]);
          stt = __shfl_sync(0xffffffffu, stt, 0);
          if (stt == 2) break;
          if (stt == 1) pf[4] += refresh_tasks(c, p, lane, pf[5], reinterpret_cast<uint32_t*>(mine));
          if (lane == 0) __nanosleep(128);
          __syncwarp();
        }
        __threadfence();
      }
      if (prof) pf[2] = gtime();
      ++pf[6];
      draft_seq(c, s, prompt_id, a.seq_tok, a.stride, a.seq_len, d.pos_base, cursor, tag,
                d.match_len, d.draft_len, d.draft_tok, d.draft_parent, d.draft_depth, d.draft_pos,
                d.draft_mask, M, merge, lane, c.pdirty);
      __syncwarp();
      uint32_t last = 0;
      if (lane == 0) {
        __threadfence();
        last = atomicAdd(c.st_ndone, 1u) + 1 == (uint32_t)n;
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        __threadfence();
        row_offsets_warp(n, d.draft_len, d.row_offsets, lane);
      }
    }
  }
  if (prof && lane == 0) {
    pf[3] = gtime();
    for (int i = 0; i < 8; ++i) prof[(size_t)gw * 8 + i] = pf[i];
  }
  (void)sh_last;
}


// ---- the tree step beside the scan (srt_cache_set_step_overlap, D <= 32;
// measured slower than the step after the scan on B200, so off by default:
// DESIGN.md §5).  The scan runs on all SMs but G; this kernel, a
// programmatic dependent launch of the scan, runs G CTAs of OV_WARPS warps
// (each fills an SM's register file) on the SMs the scan leaves, and commits
// and inserts each sequence as soon as the scan has finished that sequence's
// rows (ov.seq_done, counted by the scan's last worker of each row).  Work
// items, claimed dynamically by every warp:
//   * phase 1 of sequence s (the sequences in order, as the scan finishes
//     them): accept + cursor insert; the last of a prompt publishes its hub
//     refresh tasks (ov.rf) and starts on them;
//   * a prompt's hub refresh tasks (any warp, while it waits);
//   * the draft of one sequence whose prompt is ready (ov.dq, appended by the
//     warp that finishes the prompt's refresh).
// A warp waiting for the scan runs the other two kinds.  No wait depends on
// a warp that is not running or on the scan's completion (the scan never
// waits on this kernel), so neither co-residency nor actual overlap is
// needed for progress: run after the scan, the kernel gives the same result.
constexpr int OV_WARPS = 12;

struct OvState {
  int64_t* total;      // row_offsets[n] as of the call (the scan's row count: the caller's
                       // row_offsets may be overwritten by the next drafts meanwhile)
  uint32_t* seq_done;  // [n] rows of sequence s the scan has finished
  uint32_t* plist;     // [n] the batch's sequences grouped by prompt
  uint32_t* pstart;    // [P + 1] prompt p's sequences: plist[pstart[p] .. pstart[p + 1])
  uint32_t* pfill;     // [P] (prep scratch)
  uint32_t* dq;        // [n] draft queue (NONE until written)
  uint32_t* rf;        // [P] prompts with published refresh tasks (NONE until written)
  uint32_t* ctr;       // [0] next phase-1 sequence, [1] draft entries reserved,
                       // [2] draft entries claimed, [3] rf entries reserved
};

size_t ov_words(int32_t n, int32_t P) { return 2 + 3 * (size_t)n + 3 * (size_t)P + 1 + 8; }
OvState ov_carve(uint32_t* b, int32_t n, int32_t P) {
  OvState o;
  o.total = reinterpret_cast<int64_t*>(b);  // (the buffer is 256-byte aligned)
  o.seq_done = b + 2;
  o.plist = o.seq_done + n;
  o.dq = o.plist + n;
  o.pstart = o.dq + n;
  o.pfill = o.pstart + P + 1;
  o.rf = o.pfill + P;
  o.ctr = o.rf + P;
  return o;
}

// k_step_prep plus the overlap state: per-prompt sequence lists (a counting
// sort by prompt), cleared row counters and queues.  One CTA.
__global__ void __launch_bounds__(1024) k_step_prep_ov(DevCache c, int32_t n,
                                                       const int32_t* __restrict__ prompt_id,
                                                       const int64_t* __restrict__ row_offsets,
                                                       OvState o) {
  __shared__ uint32_t carry_sh;
  __shared__ uint32_t wsum[32];
  for (int32_t i = threadIdx.x; i < c.P; i += blockDim.x) {
    c.st_pcount[i] = 0;
    c.st_pdone[i] = 0;
    c.st_pready[i] = 0;
    c.st_pnd[i] = 0;
    c.st_pnext[i] = 0;
    c.st_pfin[i] = 0;
    o.pfill[i] = 0;
    o.rf[i] = NONE;
  }
  for (int32_t s = threadIdx.x; s < n; s += blockDim.x) {
    o.seq_done[s] = 0;
    o.dq[s] = NONE;
  }
  if (threadIdx.x < 8) o.ctr[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    *c.st_ndone = 0;
    carry_sh = 0;
    *o.total = row_offsets[n];
  }
  __syncthreads();
  for (int32_t s = threadIdx.x; s < n; s += blockDim.x) {
    const int32_t p = prompt_id[s];
    if (p >= 0 && p < c.P) atomicAdd(&c.st_pcount[p], 1u);
  }
  __syncthreads();
  // pstart = exclusive prefix sum of pcount (block scan, 1024 prompts a pass)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int32_t b = 0; b < c.P; b += blockDim.x) {
    const int32_t i = b + threadIdx.x;
    const uint32_t v = i < c.P ? c.st_pcount[i] : 0u;
    uint32_t x = v;
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, k);
      if (lane >= k) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t z = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
      for (int k = 1; k < 32; k <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, z, k);
        if (lane >= k) z += y;
      }
      wsum[lane] = z;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t carry = carry_sh;
    const uint32_t excl = carry + (w ? wsum[w - 1] : 0u) + x - v;
    if (i < c.P) o.pstart[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_sh = carry + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) o.pstart[c.P] = carry_sh;
  __syncthreads();
  for (int32_t s = threadIdx.x; s < n; s += blockDim.x) {
    const int32_t p = prompt_id[s];
    if (p >= 0 && p < c.P) o.plist[o.pstart[p] + atomicAdd(&o.pfill[p], 1u)] = (uint32_t)s;
  }
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *(const volatile uint32_t*)p;
}

template <int WPC>
__global__ void __launch_bounds__(WPC * 32, 1)
k_tree_step_ov(DevCache c, VerifyArgs a, const unsigned long long* __restrict__ result,
               const int32_t* __restrict__ prompt_id, const int32_t* __restrict__ floor_,
               uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats,
               StepDraftArgs d, OvState o) {
  extern __shared__ __align__(16) unsigned char step_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* mine = step_smem + (size_t)w * tree_step_smem_per_warp_dev(c.D);
  const int32_t n = a.n;
  const int32_t gw = blockIdx.x * WPC + w;
  unsigned long long* const prof = g_step_prof;
  unsigned long long pf[8] = {prof ? gtime() : 0ull, 0, 0, 0, 0, 0, 0, 0};

  // append sequences [b, e) of plist (or the single sequence `one`) to the
  // draft queue; the caller has fenced after everything the drafts read
  auto push_drafts = [&](const uint32_t* src, uint32_t cnt) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&o.ctr[1], cnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (uint32_t i = lane; i < cnt; i += 32)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(o.dq + base + i), "r"(src[i])
                   : "memory");
    __syncwarp();
  };
  auto push_prompt = [&](int32_t p) {
    const uint32_t b = o.pstart[p], e = o.pstart[p + 1];
    push_drafts(o.plist + b, e - b);
  };
  // one draft whose prompt is ready, if any entry is reserved and unclaimed
  auto try_draft = [&]() -> bool {
    uint32_t idx = NONE;
    if (lane == 0) {
      uint32_t h = ld_volatile_u32(&o.ctr[2]);
      while (h < ld_volatile_u32(&o.ctr[1])) {
        const uint32_t old = atomicCAS(&o.ctr[2], h, h + 1);
        if (old == h) {
          idx = h;
          break;
        }
        h = old;
      }
    }
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx == NONE) return false;
    uint32_t s = NONE;
    if (lane == 0)
      do s = ld_acquire_u32(&o.dq[idx]); while (s == NONE);
    s = __shfl_sync(0xffffffffu, s, 0);
    __threadfence();
    ++pf[6];
    draft_seq(c, (int32_t)s, prompt_id, a.seq_tok, a.stride, a.seq_len, d.pos_base, cursor, tag,
              d.match_len, d.draft_len, d.draft_tok, d.draft_parent, d.draft_depth, d.draft_pos,
              d.draft_mask, reinterpret_cast<unsigned long long*>(mine),
              reinterpret_cast<Ent*>(mine + 64 * 8), lane, c.pdirty);
    __syncwarp();
    uint32_t last = 0;
    if (lane == 0) {
      __threadfence();
      last = atomicAdd(c.st_ndone, 1u) + 1 == (uint32_t)n;
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      __threadfence();
      row_offsets_warp(n, d.draft_len, d.row_offsets, lane);
    }
    return true;
  };
  // run refresh tasks of a recently published prompt, if one has any left
  auto run_refresh = [&](int32_t p) {
    bool fin = false;
    pf[4] += refresh_tasks(c, p, lane, pf[5], reinterpret_cast<uint32_t*>(mine), &fin);
    if (fin) push_prompt(p);
  };
  auto try_refresh = [&]() -> bool {
    int32_t pick = -1;
    if (lane == 0) {
      const uint32_t t = ld_volatile_u32(&o.ctr[3]);
      for (uint32_t i = t; i > 0 && i + 8 > t; --i) {
        const uint32_t p = ld_volatile_u32(&o.rf[i - 1]);
        if (p == NONE) continue;
        if (ld_acquire_u32(&c.st_pready[p]) == 1u &&
            ld_volatile_u32(&c.st_pnext[p]) < ld_volatile_u32(&c.st_pnd[p])) {
          pick = (int32_t)p;
          break;
        }
      }
    }
    pick = __shfl_sync(0xffffffffu, pick, 0);
    if (pick < 0) return false;
    __threadfence();
    run_refresh(pick);
    return true;
  };

  bool p1_left = true;
  while (true) {
    if (try_draft()) continue;
    if (p1_left) {
      uint32_t s = 0;
      if (lane == 0) s = atomicAdd(&o.ctr[0], 1u);
      s = __shfl_sync(0xffffffffu, s, 0);
      if (s >= (uint32_t)n) {
        p1_left = false;
        continue;
      }
      // wait for the scan to finish the sequence's rows, helping meanwhile
      const uint32_t rows = (uint32_t)(a.row_offsets[s + 1] - a.row_offsets[s]);
      while (true) {
        uint32_t done = 0;
        if (lane == 0) done = ld_acquire_u32(&o.seq_done[s]);
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done >= rows) break;
        if (!try_draft() && !try_refresh() && lane == 0) __nanosleep(64);
        __syncwarp();
      }
      __threadfence();
      CursorSmem S = carve_cursor_smem(mine, 0, c.D);
      int32_t* ctok = reinterpret_cast<int32_t*>(mine + cursor_warp_bytes(c.D));
      const int32_t t = accept_seq(c, a, result, (int32_t)s, ctok, ctok + 65, lane);
      __syncwarp();
      const int32_t t_end = a.seq_len[s];
      const int32_t p = prompt_id[s];
      if (p < 0 || p >= c.P) {
        if (lane == 0) set_error(c, SRT_DEV_BAD_PROMPT);
        __threadfence();
        push_drafts(&s, 1);  // (an empty draft; s is read by lane 0 .. 0 only)
        continue;
      }
      uint32_t* const pdl = c.pdirty + (size_t)p * PDIRTY_WORDS;
      S.pdl = pdl;
      cursor_insert_seq<1>(c, S, (int32_t)s, p, t, t_end, a.seq_tok, a.stride, floor_, INT_MAX,
                           cursor, tag, stats);
      __syncwarp();
      uint32_t last = 0;
      if (lane == 0) {
        __threadfence();  // this sequence's tree updates before the prompt's count
        last = atomicAdd(&c.st_pdone[p], 1u) + 1 == c.st_pcount[p];
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        __threadfence();  // every sibling's updates (they fenced before counting)
        const uint32_t n_t = min(*(volatile uint32_t*)pdl, PDIRTY_CAP);
        const uint32_t nd = group_touches(c, p, pdl, n_t,
                                          reinterpret_cast<unsigned long long*>(mine), lane);
        if (lane == 0) {
          c.st_pnd[p] = nd;
          if (!nd) pdl[0] = 0;
          __threadfence();
          atomicExch(&c.st_pready[p], nd ? 1u : 2u);
          if (nd) {
            const uint32_t e = atomicAdd(&o.ctr[3], 1u);
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(o.rf + e), "r"((uint32_t)p)
                         : "memory");
          }
        }
        __syncwarp();
        if (nd) run_refresh(p);
        else push_prompt(p);
      }
      continue;
    }
    // no phase-1 work left: the remaining drafts wait on other warps' refreshes
    if (ld_volatile_u32(&o.ctr[2]) >= (uint32_t)n) break;
    if (!try_refresh() && lane == 0) __nanosleep(128);
    __syncwarp();
  }
  if (prof && lane == 0) {
    pf[3] = gtime();
    pf[1] = pf[2] = pf[3];
    for (int i = 0; i < 8; ++i) prof[(size_t)gw * 8 + i] = pf[i];
  }
}
}  // namespace

size_t tree_step_smem_per_warp(int32_t D) {
  const size_t per_warp = (cursor_warp_bytes(D) + 2 * 65 * 4 + 15) & ~size_t(15);
  const size_t dr = 64 * 8 + 64 * sizeof(Ent);
  return per_warp > dr ? per_warp : dr;
}

cudaError_t launch_tree_step(const DevCache& c, const VerifyArgs& a,
                             const unsigned long long* result, const int32_t* prompt_id,
                             const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                             srt_insert_stats* stats, const int32_t* pos_base, int32_t* match_len,
                             int32_t* draft_len, int32_t* draft_tok, int32_t* draft_parent,
                             int32_t* draft_depth, int32_t* draft_pos, uint64_t* draft_mask,
                             int64_t* row_offsets, cudaStream_t stream) {
  const int ng = (c.D + 31) >> 5;
  if (ng > 4) return cudaErrorInvalidValue;  // D <= SRT_CURSOR_MAX_DEPTH
  if (a.n <= 0) return cudaSuccess;
  k_step_prep<<<1, 1024, 0, stream>>>(c, a.n, prompt_id);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // SRT_TREE_GRID=<CTAs> (development knob): D <= 32 only, 12 warps per CTA
  // (one CTA fills an SM's registers), at most that many CTAs
  static int tree_grid = -1;
  if (tree_grid < 0) {
    const char* ev = getenv("SRT_TREE_GRID");
    tree_grid = ev ? atoi(ev) : 0;
  }
  const bool wide = ng == 1 && tree_grid > 0;
  const int wpc = wide ? 12 : ng == 1 ? STEP_WARPS : ng;  // warps per CTA
  const size_t smem = (size_t)wpc * tree_step_smem_per_warp(c.D);
  auto kern = wide ? k_tree_step<1, 12> : ng == 1 ? k_tree_step<1> : ng == 2 ? k_tree_step<2>
            : ng == 3 ? k_tree_step<3> : k_tree_step<4>;
  const int kslot = wide ? 0 : ng;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // every CTA resident: a draft waits on other warps' inserts
  static int per_sm[5] = {0, 0, 0, 0, 0};
  static size_t per_sm_smem[5] = {0, 0, 0, 0, 0};
  if (!per_sm[kslot] || per_sm_smem[kslot] != smem) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[kslot], kern, wpc * 32, smem);
    if (e != cudaSuccess || per_sm[kslot] <= 0)
      return e != cudaSuccess ? e : cudaErrorInvalidConfiguration;
    per_sm_smem[kslot] = smem;
  }
  const int need = ng == 1 ? (a.n + wpc - 1) / wpc : a.n;
  int grid = need < per_sm[kslot] * num_sms() ? need : per_sm[kslot] * num_sms();
  if (wide && grid > tree_grid) grid = tree_grid;
  StepDraftArgs d{pos_base, match_len, draft_len, draft_tok, draft_parent, draft_depth,
                  draft_pos, draft_mask, row_offsets};
  static int dbg = -1;
  static unsigned long long* pbuf = nullptr;
  if (dbg < 0) {
    const char* ev = getenv("SRT_STEP_PROF");
    dbg = ev ? atoi(ev) : 0;
    if (dbg) {
      cudaMalloc(&pbuf, (size_t)8 * 65536 * 8);
      cudaMemcpyToSymbol(g_step_prof, &pbuf, sizeof(pbuf));
    }
  }
  kern<<<grid, wpc * 32, smem, stream>>>(c, a, result, prompt_id, floor_, cursor, tag, stats, d);
  e = cudaGetLastError();
  if (dbg && e == cudaSuccess && grid * wpc <= 65536) {
    const int nw = grid * wpc;
    std::vector<unsigned long long> h((size_t)nw * 8);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), pbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, p1 = 0, rel = 0, end = 0, rmax = 0, rsum = 0, hubs = 0;
    double p1sum = 0, wait_sum = 0, draft_sum = 0, draft_max = 0, wait_max = 0;
    int cnt = 0, nref = 0;
    for (int i = 0; i < nw; ++i) t0 = std::min(t0, h[(size_t)i * 8]);
    for (int i = 0; i < nw; ++i) {
      const unsigned long long* q = &h[(size_t)i * 8];
      if (!q[6]) continue;
      ++cnt;
      p1 = std::max(p1, q[1] - t0);
      p1sum += q[1] - t0;
      rel = std::max(rel, q[2] - t0);
      end = std::max(end, q[3] - t0);
      wait_sum += q[2] - q[1];
      wait_max = std::max(wait_max, (double)(q[2] - q[1]));
      draft_sum += q[3] - q[2];
      draft_max = std::max(draft_max, (double)(q[3] - q[2]));
      if (q[5]) { ++nref; rsum += q[4]; rmax = std::max(rmax, q[4]); hubs += q[5]; }
    }
    unsigned long long rs[2] = {0, 0};
    cudaMemcpyFromSymbol(rs, g_refresh_stats, sizeof rs);
    fprintf(stderr, "[tree step] hub refreshes so far: %llu incremental, %llu full scans\n", rs[0],
            rs[1]);
    fprintf(stderr, "[tree step] warps %d: phase1 end max %.1f mean %.1f us; wait max %.1f mean %.1f us; "
            "release max %.1f us; draft max %.1f mean %.1f us; end %.1f us; refreshes %d (%llu hubs) "
            "max %.1f mean %.1f kcycles\n",
            cnt, p1 / 1e3, p1sum / cnt / 1e3, wait_max / 1e3, wait_sum / cnt / 1e3, rel / 1e3,
            draft_max / 1e3, draft_sum / cnt / 1e3, end / 1e3, nref, hubs, rmax / 1e3,
            nref ? rsum / 1e3 / nref : 0.0);
  }
  return e;
}

size_t tree_step_ov_words(int32_t n, int32_t P) { return ov_words(n, P); }

cudaError_t launch_step_prep_ov(const DevCache& c, int32_t n, const int32_t* prompt_id,
                                const int64_t* row_offsets, uint32_t* ovbuf, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  k_step_prep_ov<<<1, 1024, 0, stream>>>(c, n, prompt_id, row_offsets, ov_carve(ovbuf, n, c.P));
  return cudaGetLastError();
}

uint32_t* tree_step_ov_seq_done(uint32_t* ovbuf, int32_t n, int32_t P) {
  return ov_carve(ovbuf, n, P).seq_done;
}

const int64_t* tree_step_ov_total(uint32_t* ovbuf, int32_t n, int32_t P) {
  return ov_carve(ovbuf, n, P).total;
}

cudaError_t launch_tree_step_ov(const DevCache& c, const VerifyArgs& a,
                                const unsigned long long* result, const int32_t* prompt_id,
                                const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                                srt_insert_stats* stats, const int32_t* pos_base,
                                int32_t* match_len, int32_t* draft_len, int32_t* draft_tok,
                                int32_t* draft_parent, int32_t* draft_depth, int32_t* draft_pos,
                                uint64_t* draft_mask, int64_t* row_offsets, uint32_t* ovbuf,
                                int grid, cudaStream_t stream) {
  if (c.D > 32 || grid <= 0) return cudaErrorInvalidValue;
  if (a.n <= 0) return cudaSuccess;
  const size_t smem = (size_t)OV_WARPS * tree_step_smem_per_warp(c.D);
  auto kern = k_tree_step_ov<OV_WARPS>;
  static size_t set_smem = 0;
  if (set_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  StepDraftArgs d{pos_base, match_len, draft_len, draft_tok, draft_parent, draft_depth,
                  draft_pos, draft_mask, row_offsets};
  // a programmatic dependent launch: it may start once every CTA of the scan
  // before it has triggered (they do as they start), on the SMs the scan left
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(OV_WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c, a, result, prompt_id, floor_, cursor, tag, stats, d,
                            ov_carve(ovbuf, a.n, c.P));
}

}  // namespace srt
