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

constexpr int PLAN_THREADS = 1024;

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
              const int32_t* __restrict__ floor_, long long* __restrict__ offs) {
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
      long long t = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
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
  while ((uint32_t)(v = ld_acquire_u64(&s->val)) == NONE) __nanosleep(32);
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

}  // namespace

cudaError_t launch_insert_plan(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* from, const int32_t* to, const int32_t* floor_,
                               long long* scratch, cudaStream_t stream) {
  k_insert_plan<<<1, PLAN_THREADS, 0, stream>>>(c, n, prompt_id, from, to, floor_, scratch);
  return cudaGetLastError();
}

cudaError_t launch_insert_walk(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* seq_tok, int64_t stride, const int32_t* from,
                               const int32_t* to, const int32_t* floor_, srt_insert_stats* stats,
                               const long long* scratch, cudaStream_t stream) {
  k_insert_walk<<<num_sms() * 8, 256, 0, stream>>>(c, n, prompt_id, seq_tok, stride, from, to,
                                                   floor_, scratch, stats);
  return cudaGetLastError();
}

}  // namespace srt
