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
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int PLAN_THREADS = 256;  // small: co-resides with a running verify scan

__device__ __forceinline__ int32_t span_lo(int32_t from, int32_t floor_, int32_t D) {
  int32_t lo = from - D + 1;
  if (lo < floor_) lo = floor_;
  if (lo < 0) lo = 0;
  return lo;
}

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

// Warp-aggregated id allocation from a bump counter.  Returns BAD when the
// pool is exhausted.
__device__ __forceinline__ uint32_t bump_alloc(unsigned long long* ctr, unsigned long long amount,
                                               unsigned long long limit) {
  const unsigned m = __activemask();
  const int leader = __ffs(m) - 1;
  const int lane = threadIdx.x & 31;
  // every active lane asks for the same `amount` here (1 node id)
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, amount * (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  const unsigned long long id = base + amount * (unsigned long long)__popc(m & lanemask_lt());
  return (id + amount <= limit) ? (uint32_t)id : BAD;
}

// One 16-byte relaxed load of a hash slot: key and (val, aux) together, so
// the common case (an existing edge) costs one round trip per hop.
__device__ __forceinline__ void ld_slot(const HashSlot* s, unsigned long long& key,
                                        uint32_t& val, uint32_t& aux) {
  unsigned long long k, v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(v) : "l"(s)
               : "memory");
  key = k;
  val = (uint32_t)v;
  aux = (uint32_t)(v >> 32);
}

// Probe for `key`; if absent, claim the first EMPTY slot with a CAS.
// Returns the slot index (or -1 if the table is full); *created tells whether
// this thread inserted the key (its value is then still NONE = pending);
// *val / *aux are the slot's words as read (val NONE if pending or created).
__device__ __forceinline__ long long hash_acquire(const DevCache& c, unsigned long long key,
                                                  bool* created, uint32_t* val, uint32_t* aux) {
  const unsigned long long mask = c.H - 1;
  unsigned long long h = mix64(key) & mask;
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    HashSlot* s = c.hash + h;
    unsigned long long k;
    uint32_t v, a;
    ld_slot(s, k, v, a);
    if (k == EMPTY_KEY) {
      k = atomicCAS(&s->key, EMPTY_KEY, key);
      if (k == EMPTY_KEY) {
        *created = true;
        *val = NONE;
        *aux = NONE;
        return (long long)h;
      }
      v = NONE;  // another thread claimed this slot: re-read its value later
    }
    if (k == key) {
      *created = false;
      *val = v;
      *aux = a;
      return (long long)h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

// Wait for a pending slot's publication; returns val, *aux gets aux.
__device__ __forceinline__ uint32_t wait_value(const HashSlot* s, uint32_t* aux) {
  unsigned long long v;
  while ((uint32_t)(v = ld_relaxed_u64((const unsigned long long*)&s->val)) == NONE) __nanosleep(32);
  *aux = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// Wait until block i of node u has been published (its unique creator is the
// thread that claimed slot blk_start(i)).
__device__ uint32_t wait_block(const DevCache& c, uint32_t u, uint32_t i) {
  const unsigned long long key = block_key(u, i);
  const unsigned long long mask = c.H - 1;
  while (true) {
    unsigned long long h = mix64(key) & mask;
    for (unsigned long long probe = 0; probe <= mask; ++probe) {
      HashSlot* s = c.hash + h;
      const unsigned long long k = ld_relaxed_u64(&s->key);
      uint32_t unused;
      if (k == key) return wait_value(s, &unused);
      if (k == EMPTY_KEY) break;
      h = (h + 1) & mask;
    }
    __nanosleep(64);
    if (ld_acquire_u32(c.status) & SRT_DEV_CAPACITY) return BAD;
  }
}

// Append child `ch` (token tk) to node u's children.  Child 0 lives inline in
// rec[u]; child k >= 1 goes to slot k-1 of the geometric blocks, each created
// by the thread that claims its first slot and published through the hash.
// Returns the child's slot word (NONE for the inline child 0, BAD on failure).
__device__ uint32_t attach_child(const DevCache& c, uint32_t u, uint32_t ch, int32_t tk) {
  const uint32_t k0 = atomicAdd(&c.rec[u].x, 1u);
  if (k0 == 0) {  // read only by later kernels
    c.rec[u].y = ch;
    c.rec[u].z = (uint32_t)tk;
    return NONE;
  }
  const uint32_t k = k0 - 1;
  const uint32_t i = blk_index(k);
  const uint32_t off = k - blk_start(i);
  uint32_t base;
  if (off == 0) {  // this thread creates block i
    const uint32_t sz = blk_size(i);
    const unsigned long long b = atomicAdd(&c.ctr[1], (unsigned long long)sz);
    base = (b + sz <= c.W) ? (uint32_t)b : BAD;
    if (base == BAD) set_error(c, SRT_DEV_CAPACITY);
    bool created = false;
    uint32_t unused, unused2;
    const long long h = hash_acquire(c, block_key(u, i), &created, &unused, &unused2);
    if (h < 0) {
      set_error(c, SRT_DEV_CAPACITY);
      return BAD;  // waiters poll the status word
    }
    publish_slot(c.hash + h, base, NONE);
  } else {
    base = wait_block(c, u, i);
  }
  if (base == BAD) return BAD;
  c.slots[base + off] = ch;
  c.stok[base + off] = tk;
  return base + off;
}

// Child of u labelled tk, created if missing; *pos = its slot word (NONE for
// an inline child 0).  BAD if a pool is exhausted.
__device__ __forceinline__ uint32_t get_or_create(const DevCache& c, uint32_t u, int32_t tk,
                                                  uint32_t* pos, unsigned& created_ctr) {
  bool created = false;
  uint32_t v = NONE;
  const long long h = hash_acquire(c, edge_key(u, (uint32_t)tk), &created, &v, pos);
  if (h < 0) {
    set_error(c, SRT_DEV_CAPACITY);
    return BAD;
  }
  HashSlot* s = c.hash + h;
  if (!created) return v != NONE ? v : wait_value(s, pos);
  const uint32_t id = bump_alloc(&c.ctr[0], 1, c.N);
  if (id == BAD) {
    set_error(c, SRT_DEV_CAPACITY);
    publish_slot(s, BAD, NONE);
    return BAD;
  }
  c.tok[id] = tk;
  *pos = attach_child(c, u, id, tk);
  publish_slot(s, id, *pos);
  ++created_ctr;
  return id;
}

// get_or_create for a whole warp in lockstep (every lane calls it; inactive
// lanes return BAD): the lanes that claimed a new edge take their node ids
// with ONE atomic per warp, so the id counter sees 1/32 of the traffic.
__device__ __forceinline__ uint32_t get_or_create_warp(const DevCache& c, bool active, uint32_t u,
                                                       int32_t tk, uint32_t* pos,
                                                       unsigned& created_ctr) {
  bool created = false;
  uint32_t v = NONE;
  long long h = -1;
  *pos = NONE;
  if (active) {
    h = hash_acquire(c, edge_key(u, (uint32_t)tk), &created, &v, pos);
    if (h < 0) set_error(c, SRT_DEV_CAPACITY);
  }
  const unsigned need = __ballot_sync(0xffffffffu, created);
  unsigned long long base = 0;
  if (need) {
    const int leader = __ffs(need) - 1;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(&c.ctr[0], (unsigned long long)__popc(need));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  if (!active || h < 0) return BAD;
  HashSlot* s = c.hash + h;
  if (!created) return v != NONE ? v : wait_value(s, pos);
  const unsigned long long idl = base + __popc(need & lanemask_lt());
  if (idl + 1 > c.N) {
    set_error(c, SRT_DEV_CAPACITY);
    publish_slot(s, BAD, NONE);
    return BAD;
  }
  const uint32_t id = (uint32_t)idl;
  c.tok[id] = tk;
  *pos = attach_child(c, u, id, tk);
  publish_slot(s, id, *pos);
  ++created_ctr;
  return id;
}

__global__ void __launch_bounds__(256)
k_insert_walk(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
              const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ from,
              const int32_t* __restrict__ to, const int32_t* __restrict__ floor_,
              const long long* __restrict__ offs, srt_insert_stats* stats) {
  const long long total = offs[n];
  unsigned windows = 0, incs = 0, created = 0;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    // span s: offs[s] <= idx < offs[s+1]
    int32_t lo_s = 0, hi_s = n - 1;
    while (lo_s < hi_s) {
      const int32_t mid = (lo_s + hi_s + 1) >> 1;
      if (offs[mid] <= idx) lo_s = mid; else hi_s = mid - 1;
    }
    const int32_t s = lo_s;
    const int32_t f = from[s], t_end = to[s];
    const int32_t i = span_lo(f, floor_ ? floor_[s] : 0, c.D) + (int32_t)(idx - offs[s]);
    const int32_t* toks = seq_tok + (int64_t)s * stride;
    uint32_t u = (uint32_t)prompt_id[s];
    const int32_t end = min(i + c.D, t_end);
    ++windows;
    for (int32_t j = i; j < end; ++j) {
      const int32_t tk = toks[j];
      if (tk < 0 || tk >= c.V) {
        set_error(c, SRT_DEV_OOV);
        break;
      }
      uint32_t pos;
      const uint32_t ch = get_or_create(c, u, tk, &pos, created);
      if (ch >= BAD) break;
      if (j >= f) {  // a window ends at a new position: count it (and its parent's csum)
        atomicAdd(&c.cnt[ch], 1u);
        if (pos < BAD) atomicAdd(&c.scnt[pos], 1u);
        atomicAdd(&c.rec[u].w, 1u);
        ++incs;
      }
      u = ch;
    }
  }
  if (stats) {
    unsigned long long a = windows, b = incs, d = created;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if ((threadIdx.x & 31) == 0 && (a | b | d)) {
      atomicAdd(&stats->windows, a);
      atomicAdd(&stats->increments, b);
      atomicAdd(&stats->nodes_created, d);
    }
  }
}

// ---------------------------------------------------------------------------
// Cursor insertion (srt_insert_cursor).  A sequence's cursor at position P
// holds A_l = node(y[P-l .. P-1]) for l = 1..D (the suffix nodes).  Appending
// y_P: A'_1 = child(root, y_P), A'_l = child(A_{l-1}, y_P), and every A'_l
// (l <= min(D, P - floor + 1)) is exactly the node of a window ending at P, so
// it gets +1.  That is one hop per window end instead of a root walk, and the
// D hops of a position run in parallel across the lanes of the sequence's
// warp.  An invalid cursor is rebuilt by walking the D-1 suffixes from the
// root, which creates precisely the nodes the walk kernel creates for window
// starts before P (uncounted), so both kernels build the same tree.
// Cursor record (u32 words): [0] cache tag, [1] P, [2] prompt, [3] floor,
// [4 .. 4+D) A_1 .. A_D (NONE = no node).
// ---------------------------------------------------------------------------
constexpr int CURSOR_WARPS = 4;

// Development-only per-sequence profile (srt_debug_insert_profile): when set,
// k_insert_cursor writes {total cycles, cursor-phase cycles, positions, nodes
// created, slowest position's cycles, cursor valid, 0, 0} per sequence.
__device__ long long* g_ins_prof = nullptr;

__global__ void __launch_bounds__(CURSOR_WARPS * 32)
k_insert_cursor(DevCache c, int32_t n, const int32_t* __restrict__ prompt_id,
                const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ from,
                const int32_t* __restrict__ to, const int32_t* __restrict__ floor_, int32_t short_max,
                uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  extern __shared__ uint32_t cur_smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * CURSOR_WARPS + w;
  if (s >= n) return;
  const int32_t D = c.D;
  uint32_t* A = cur_smem + (size_t)w * (D + 1);  // A[l], l = 1..D; A[0] = root
  uint32_t* cur = cursor + (size_t)s * (D + 4);
  const int32_t p = prompt_id[s];
  if (p < 0 || p >= c.P) return;  // flagged by the plan kernel
  const int32_t f = from[s], t_end = to[s];
  const int32_t fl = floor_ ? floor_[s] : 0;
  const int32_t P = max(f, fl);
  if (t_end <= P) return;  // no window ends at a new position: cursor untouched
  if (t_end - P > short_max) {  // long span: the walk kernel inserts it
    if (lane == 0) cur[1] = NONE;  // and the cursor must be rebuilt next time
    return;
  }
  const int32_t* y = seq_tok + (int64_t)s * stride;
  const long long tp0 = clock64();
  long long tp_cur = 0, tp_max = 0;
  unsigned incs = 0, created = 0;
  const bool valid = cur[0] == tag && cur[1] == (uint32_t)P && cur[2] == (uint32_t)p &&
                     cur[3] == (uint32_t)fl;
  if (lane == 0) A[0] = (uint32_t)p;
  if (valid) {
    for (int32_t l = 1 + lane; l <= D; l += 32) A[l] = cur[4 + l - 1];
  } else {
    // rebuild: A_l for l <= min(D-1, P-floor) by walking y[P-l .. P-1] from the
    // root (creating missing nodes, counting nothing: these windows end < P)
    const int32_t lmax = min(D - 1, P - max(fl, 0));
    for (int32_t l = 1 + lane; l <= D; l += 32) {
      uint32_t u = NONE;
      if (l <= lmax) {
        u = (uint32_t)p;
        for (int32_t j = P - l; j < P; ++j) {
          const int32_t tk = y[j];
          if (tk < 0 || tk >= c.V) {
            set_error(c, SRT_DEV_OOV);
            u = NONE;
            break;
          }
          uint32_t pos;
          u = get_or_create(c, u, tk, &pos, created);
          if (u >= BAD) {
            u = NONE;
            break;
          }
        }
      }
      A[l] = u;
    }
  }
  __syncwarp();
  tp_cur = clock64() - tp0;
  const int ngroups = (D + 31) >> 5;
  for (int32_t j = P; j < t_end; ++j) {
    const long long tj = clock64();
    const int32_t tk = y[j];
    const bool oov = tk < 0 || tk >= c.V;
    if (oov && lane == 0) set_error(c, SRT_DEV_OOV);
    const int32_t lim = min(D, j - max(fl, 0) + 1);  // windows ending at j start >= floor
    // descending groups: group g reads A[32g .. 32g+31] (old) before group g-1
    // overwrites A[32g - 32 + 1 .. 32g]
    for (int g = ngroups - 1; g >= 0; --g) {
      const int32_t l = 32 * g + lane + 1;
      uint32_t par = NONE;
      if (l <= D) par = A[l - 1];
      __syncwarp();
      const bool active = l <= D && !oov && l <= lim && par < BAD;
      uint32_t pos;
      const uint32_t ch = get_or_create_warp(c, active, par, tk, &pos, created);
      if (active && ch < BAD) {
        atomicAdd(&c.cnt[ch], 1u);
        if (pos < BAD) atomicAdd(&c.scnt[pos], 1u);
        atomicAdd(&c.rec[par].w, 1u);
        ++incs;
      }
      if (l <= D) A[l] = (active && ch < BAD) ? ch : NONE;
      __syncwarp();
    }
    tp_max = max(tp_max, clock64() - tj);
  }
  for (int32_t l = 1 + lane; l <= D; l += 32) cur[4 + l - 1] = A[l];
  if (lane == 0) {
    cur[0] = tag;
    cur[1] = (uint32_t)t_end;
    cur[2] = (uint32_t)p;
    cur[3] = (uint32_t)fl;
  }
  if (g_ins_prof) {
    unsigned long long d = created;
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) {
      long long* o = g_ins_prof + 8 * (int64_t)s;
      o[0] = clock64() - tp0;
      o[1] = tp_cur;
      o[2] = t_end - P;
      o[3] = (long long)d;
      o[4] = tp_max;
      o[5] = valid;
    }
  }
  if (stats) {
    unsigned long long b = incs, d = created;
    for (int o = 16; o; o >>= 1) {
      b += __shfl_xor_sync(0xffffffffu, b, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
    }
    if (lane == 0) {
      // window starts the walk kernel would have walked for this span
      const int32_t lo = span_lo(f, fl, D);
      atomicAdd(&stats->windows, (unsigned long long)(t_end - lo));
      atomicAdd(&stats->increments, b);
      if (d) atomicAdd(&stats->nodes_created, d);
    }
  }
}

}  // namespace

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
  carveout_once<k_insert_walk>();
  k_insert_walk<<<num_sms() * 8, 256, 0, stream>>>(c, n, prompt_id, seq_tok, stride, from, to,
                                                   floor_, scratch, stats);
  return cudaGetLastError();
}

size_t insert_cursor_smem(int32_t D) { return (size_t)CURSOR_WARPS * (D + 1) * 4; }

cudaError_t launch_insert_cursor(const DevCache& c, int32_t n, const int32_t* prompt_id,
                                 const int32_t* seq_tok, int64_t stride, const int32_t* from,
                                 const int32_t* to, const int32_t* floor_, int32_t short_max,
                                 uint32_t* cursor, uint32_t tag, srt_insert_stats* stats,
                                 cudaStream_t stream) {
  const size_t smem = insert_cursor_smem(c.D);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_insert_cursor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  carveout_once<k_insert_cursor>();
  k_insert_cursor<<<(n + CURSOR_WARPS - 1) / CURSOR_WARPS, CURSOR_WARPS * 32, smem, stream>>>(
      c, n, prompt_id, seq_tok, stride, from, to, floor_, short_max, cursor, tag, stats);
  return cudaGetLastError();
}

}  // namespace srt
