// insert.cuh — the cursor insertion of one sequence by one warp (or NG warps)
// and the hash / child-list machinery under it, shared by the insert kernels
// (insert.cu) and the fused tree step (step.cu).  See insert.cu for the design.
#pragma once
#include "srt_internal.cuh"

namespace srt {
namespace {

__device__ __forceinline__ int32_t span_lo(int32_t from, int32_t floor_, int32_t D) {
  int32_t lo = from - D + 1;
  if (lo < floor_) lo = floor_;
  if (lo < 0) lo = 0;
  return lo;
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
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Slots h, h+1 (h even: one aligned 32-byte load): keys and aux words.
struct SlotPair {
  unsigned long long k0, k1;
  uint32_t a0, a1;
};
__device__ __forceinline__ SlotPair ld_pair(const HashSlot* s) {
  unsigned long long k0, v0, k1, v1;
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(k0), "=l"(v0), "=l"(k1), "=l"(v1)
               : "l"(s)
               : "memory");
  return SlotPair{k0, k1, (uint32_t)(v0 >> 32), (uint32_t)(v1 >> 32)};
}

// One probe step at slot h whose key was read as k (aux a): claim it if EMPTY.
// Returns 1 = created here, 2 = found here (*aux = a, NONE if unknown), 0 = go on.
__device__ __forceinline__ int probe_step(const DevCache& c, unsigned long long key,
                                          unsigned long long h, unsigned long long k, uint32_t a,
                                          uint32_t* aux) {
  if (k == EMPTY_KEY) {
    k = atomicCAS(&c.hash[h].key, EMPTY_KEY, key);
    if (k == EMPTY_KEY) {
      *aux = NONE;
      return 1;
    }
    a = NONE;  // another thread claimed this slot: its aux is not known yet
  }
  if (k == key) {
    *aux = a;
    return 2;
  }
  return 0;
}

// Probe for `key` from slot h on (two slots per load from an even slot); if
// absent, claim the first EMPTY slot with a CAS.  Returns the slot index (=
// the node id for an edge key; -1 if the table is full); *created tells
// whether this thread inserted the key; *aux is the slot's aux word as read
// (NONE if pending, created or unknown).
__device__ __forceinline__ long long hash_acquire_from(const DevCache& c, unsigned long long key,
                                                       unsigned long long h, bool* created,
                                                       uint32_t* aux) {
  const unsigned long long mask = c.H - 1;
  for (unsigned long long probe = 0; probe <= mask;) {
    if ((h & 1) == 0) {
      const SlotPair q = ld_pair(c.hash + h);
      int r = probe_step(c, key, h, q.k0, q.a0, aux);
      if (r) {
        *created = r == 1;
        return (long long)h;
      }
      r = probe_step(c, key, h + 1, q.k1, q.a1, aux);
      if (r) {
        *created = r == 1;
        return (long long)(h + 1);
      }
      h = (h + 2) & mask;
      probe += 2;
    } else {
      unsigned long long k;
      uint32_t v, a;
      ld_slot(c.hash + h, k, v, a);
      const int r = probe_step(c, key, h, k, a, aux);
      if (r) {
        *created = r == 1;
        return (long long)h;
      }
      h = (h + 1) & mask;
      probe += 1;
    }
  }
  return -1;
}
__device__ __forceinline__ long long hash_acquire(const DevCache& c, unsigned long long key,
                                                  bool* created, uint32_t* aux) {
  return hash_acquire_from(c, key, home_slot(c, key), created, aux);
}

// Wait for an edge slot's aux word (its creator publishes it after attaching).
__device__ __forceinline__ uint32_t wait_aux(const DevCache& c, uint32_t h) {
  uint32_t a;
  while ((a = ld_relaxed_u32(&c.hash[h].aux)) == NONE) {
    __nanosleep(32);
    if (ld_acquire_u32(c.status) & SRT_DEV_CAPACITY) return BAD;
  }
  return a;
}

// Wait until block i >= 4 of node u has been published in the hash (its unique
// creator is the thread that claimed slot blk_start(i)).
__device__ uint32_t wait_block(const DevCache& c, uint32_t u, uint32_t i) {
  const unsigned long long key = block_key(u, i);
  const unsigned long long mask = c.H - 1;
  while (true) {
    unsigned long long h = home_slot(c, key);
    for (unsigned long long probe = 0; probe <= mask; ++probe) {
      HashSlot* s = c.hash + h;
      const unsigned long long k = ld_relaxed_u64(&s->key);
      if (k == key) {
        uint32_t v;
        while ((v = ld_relaxed_u32(&s->val)) == NONE) __nanosleep(32);
        return v;
      }
      if (k == EMPTY_KEY) break;
      h = (h + 1) & mask;
    }
    __nanosleep(64);
    if (ld_acquire_u32(c.status) & SRT_DEV_CAPACITY) return BAD;
  }
}

// Wait until block i < 4 of node u has its base in u's record.
__device__ uint32_t wait_rec_base(const DevCache& c, uint32_t u, uint32_t i) {
  uint32_t b;
  while ((b = ld_relaxed_u32(rec_bases(c, u) + i)) == 0) {
    __nanosleep(32);
    if (ld_acquire_u32(c.status) & SRT_DEV_CAPACITY) return BAD;
  }
  return b - 1;
}

// Append child `ch` (token tk) to node u's children.  Child 0 lives inline in
// u's record; child k >= 1 goes to slot k-1 of the geometric blocks, each
// created by the thread that claims its first slot and published in u's record
// (blocks 0..3) or the hash (blocks >= 4).  Returns the child's slot word
// (AUX_CHILD0 for the inline child 0, BAD on failure).
// Child k >= 1 of u (slot k - 1 = j): create or wait for its block, fill the slot.
__device__ uint32_t place_child(const DevCache& c, uint32_t u, uint32_t k, uint32_t ch, int32_t tk);

__device__ uint32_t attach_child(const DevCache& c, uint32_t u, uint32_t ch, int32_t tk) {
  uint4* r = rec_of(c, u);
  const uint32_t k0 = atomicAdd(&r->x, 1u);
  if (k0 == 0) {  // read only by later kernels
    r->y = ch;
    r->z = (uint32_t)tk;
    return AUX_CHILD0;
  }
  return place_child(c, u, k0 - 1, ch, tk);
}

__device__ uint32_t place_child(const DevCache& c, uint32_t u, uint32_t k, uint32_t ch, int32_t tk) {
  const uint32_t i = blk_index(k);
  const uint32_t off = k - blk_start(i);
  uint32_t base;
  if (off == 0 && i < 4) {  // (a block pruning left behind is reused)
    const uint32_t old = ld_relaxed_u32(rec_bases(c, u) + i);
    if (old != 0) {
      if (old - 1 >= BAD) return BAD;
      c.slots[old - 1] = ch;
      c.stok[old - 1] = tk;
      return old - 1;
    }
  }
  if (off == 0 && i >= 4) {
    const uint32_t hb = hash_slot(c, block_key(u, i));
    if (hb != NONE) {  // left behind by pruning: reuse
      uint32_t v;
      while ((v = ld_relaxed_u32(&c.hash[hb].val)) == NONE) __nanosleep(32);
      if (v >= BAD) return BAD;
      c.slots[v] = ch;
      c.stok[v] = tk;
      return v;
    }
  }
  if (off == 0) {  // this thread creates block i
    const uint32_t sz = blk_size(i);
    const unsigned long long b = atomicAdd(&c.ctr[1], (unsigned long long)sz);
    base = (b + sz <= c.W) ? (uint32_t)b : BAD;
    if (base == BAD) set_error(c, SRT_DEV_CAPACITY);
    if (i < 4) {
      st_relaxed_u32(rec_bases(c, u) + i, base + 1u);  // BAD + 1 = NONE: failure
    } else {
      bool created = false;
      uint32_t unused;
      const long long h = hash_acquire(c, block_key(u, i), &created, &unused);
      if (h < 0) {
        set_error(c, SRT_DEV_CAPACITY);
        return BAD;  // waiters poll the status word
      }
      if (!created) {  // a block pruning left behind: reuse it (this block is not needed)
        uint32_t v;
        while ((v = ld_relaxed_u32(&c.hash[h].val)) == NONE) __nanosleep(32);
        base = v;
        if (base >= BAD) return BAD;
        c.slots[base] = ch;
        c.stok[base] = tk;
        return base;
      }
      publish_slot(c.hash + h, base, NONE);
    }
  } else {
    base = i < 4 ? wait_rec_base(c, u, i) : wait_block(c, u, i);
  }
  if (base >= BAD) return BAD;
  c.slots[base + off] = ch;
  c.stok[base + off] = tk;
  return base + off;
}

__device__ __forceinline__ bool is_slot_word(uint32_t pos) { return pos < AUX_CHILD0; }

// Child of u labelled tk, created (and attached) if missing; *pos = its slot
// word (AUX_CHILD0 for an inline child 0).  Returns the child's id, BAD if the
// table is full.
__device__ __forceinline__ uint32_t get_or_create(const DevCache& c, uint32_t u, int32_t tk,
                                                  uint32_t* pos, unsigned& created_ctr) {
  bool created = false;
  uint32_t a = NONE;
  const long long h = hash_acquire(c, edge_key(u, (uint32_t)tk), &created, &a);
  if (h < 0) {
    set_error(c, SRT_DEV_CAPACITY);
    return BAD;
  }
  const uint32_t id = (uint32_t)h;
  if (!created) {
    *pos = a != NONE ? a : wait_aux(c, id);
    return id;
  }
  c.tok[id] = tk;
  *pos = attach_child(c, u, id, tk);
  st_relaxed_u32(&c.hash[id].aux, *pos);
  ++created_ctr;
  return id;
}

// Resolve the edge keys key[g] of the lanes' active probes (creating the
// missing edges): hnew = the child's id (its slot), cre = this lane created
// it, aux = its slot word as read (NONE if unknown or pending).  A lane whose
// table is full ends with act = false and hnew = BAD.  Warp-collective.
template <int NG>
__device__ __forceinline__ int probe_edges(const DevCache& c, const unsigned long long (&key)[NG],
                                           bool (&act)[NG], uint32_t (&hnew)[NG],
                                           bool (&cre)[NG], uint32_t (&aux)[NG]) {
  const int lane = threadIdx.x & 31;
  (void)lane;
  const unsigned long long mask = c.H - 1;
  int rounds = 0;
  // Probe every depth's edge as a warp-convergent state machine: in each
  // round every unresolved probe issues its next memory operation (a slot
  // pair load and/or a CAS) before any result is used, so a position costs
  // max-over-lanes probe rounds instead of the sum of divergent paths.
  // Round 0 claims the home slot with a CAS while loading the home pair.
  // Each load reads 4 consecutive slots (two 32-byte loads) so that an
  // occupied home almost never costs more than one extra round (the CAS at
  // the first EMPTY slot seen).
  SlotPair qa[NG], qb[NG];
  unsigned long long ps[NG], cs[NG], rk[NG];
  int op[NG];  // bit 0: load slots ps .. ps+3, bit 1: CAS at cs; 0 = resolved
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    cre[g] = false;
    hnew[g] = NONE;
    aux[g] = NONE;
    op[g] = 0;
    if (!act[g]) continue;
    ps[g] = cs[g] = home_slot(c, key[g]);
    op[g] = 3;
  }
  for (int round = 0;; ++round) {
    bool live = false;
#pragma unroll
    for (int g = 0; g < NG; ++g) live |= op[g] != 0;
    if (!__any_sync(0xffffffffu, live)) break;
    ++rounds;
#pragma unroll
    for (int g = 0; g < NG; ++g) {  // issue
      if (op[g] & 1) {
        qa[g] = ld_pair(c.hash + ps[g]);
        qb[g] = ld_pair(c.hash + ((ps[g] + 2) & mask));
      }
      if (op[g] & 2) rk[g] = atomicCAS(&c.hash[cs[g]].key, EMPTY_KEY, key[g]);
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {  // resolve (registers only)
      if (!op[g]) continue;
      int from = 0;  // index among the 4 loaded slots to scan from
      if (op[g] & 2) {
        const int ci = (int)((cs[g] - ps[g]) & mask);  // 0..3: the CAS slot
        if (rk[g] == EMPTY_KEY) {
          op[g] = 0;
          cre[g] = true;
          hnew[g] = (uint32_t)cs[g];
          continue;
        }
        if (rk[g] == key[g]) {
          op[g] = 0;
          hnew[g] = (uint32_t)cs[g];
          const SlotPair& qq = ci < 2 ? qa[g] : qb[g];
          const unsigned long long kk = (ci & 1) ? qq.k1 : qq.k0;
          aux[g] = kk == key[g] ? ((ci & 1) ? qq.a1 : qq.a0) : NONE;
          continue;
        }
        from = ci + 1;  // slot cs holds another key
      }
      int next = 0;  // -1: found, 2: CAS slot ps + i, 0: load the next 4 slots
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < from || next) continue;
        const SlotPair& qq = i < 2 ? qa[g] : qb[g];
        const unsigned long long kk = (i & 1) ? qq.k1 : qq.k0;
        if (kk == key[g]) {
          hnew[g] = (uint32_t)((ps[g] + i) & mask);
          aux[g] = (i & 1) ? qq.a1 : qq.a0;
          next = -1;
        } else if (kk == EMPTY_KEY) {
          cs[g] = (ps[g] + i) & mask;
          next = 2;
        }
      }
      if (next == -1) {
        op[g] = 0;
      } else if (next == 2) {
        op[g] = 2;
      } else {
        ps[g] = (ps[g] + 4) & mask;
        cs[g] = ps[g];
        op[g] = 1;
      }
      if (round > 1 << 20) {  // never: the table would be full
        op[g] = 0;
        act[g] = false;
        hnew[g] = BAD;
        set_error(c, SRT_DEV_CAPACITY);
      }
    }
  }
  return rounds;
}

// Nodes created by this warp join the node count; more than N is a capacity
// error (the count, unlike ids, is deterministic).
__device__ __forceinline__ void count_created(const DevCache& c, unsigned created) {
  unsigned long long d = created;
  for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0 && d) {
    const unsigned long long before = atomicAdd(&c.ctr[0], d);
    if (before + d > c.N) set_error(c, SRT_DEV_CAPACITY);
  }
}

// ---------------------------------------------------------------------------
// Cursor insertion (srt_insert_cursor).  A sequence's cursor at position P
// holds A_l = node(y[P-l .. P-1]) for l = 1..D (the suffix nodes).  Appending
// y_P: A'_1 = child(root, y_P), A'_l = child(A_{l-1}, y_P), and every A'_l
// (l <= min(D, P - floor + 1)) is exactly the node of a window ending at P, so
// it gets +1.  That is one hop per window end instead of a root walk; the D
// hops of a position are independent (lane l handles depths l+1, l+33, ...,
// their probes in flight together).
//
// The only dependent work per position is the probe (or, for the child of a
// node this warp just created, a CAS straight at the home slot): a node's id is
// its hash slot, so the next position can use it at once.  Counts are
// fire-and-forget atomics.  What needs a created node's place among its
// parent's children -- linking it (nchild atomic, child-block creation) and
// the slot-mirror count -- is logged and done in a batch after the positions,
// all entries in parallel; so is the mirror count of a node another warp
// created and has not linked yet.  An invalid cursor is rebuilt by walking the
// D-1 suffixes from the root, which creates precisely the nodes the walk
// kernel creates for window starts before P (uncounted), so both kernels build
// the same tree.
// Cursor record (u32 words): [0] cache tag, [1] P, [2] prompt, [3] floor,
// [4 .. 4+D) A_1 .. A_D (NONE = no node).
// ---------------------------------------------------------------------------
constexpr int CURSOR_WARPS = 4;
constexpr int LOGCAP = 512;  // logged entries per warp before a batch flush
constexpr int MAXG = 4;      // depth groups per lane (D <= 128 = SRT_CURSOR_MAX_DEPTH)
static_assert(32 * MAXG == SRT_CURSOR_MAX_DEPTH, "cursor depth groups");

// Development-only per-sequence profile (srt_debug_insert_profile): when set,
// k_insert_cursor writes {total cycles, cursor-phase cycles, positions, nodes
// created, slowest position's cycles, cursor valid, batch cycles, 0} per sequence.
__device__ long long* g_ins_prof = nullptr;

struct CursorSmem {
  uint32_t* A;        // [D + 1] suffix node ids (A[0] = the root)
  uint8_t* fresh;     // [D + 1] created by this warp in this launch
  uint32_t* log_h;    // [LOGCAP] created nodes ...
  uint32_t* log_par;  // [LOGCAP] ... their parents
  int32_t* log_tok;   // [LOGCAP] ... their tokens
  uint32_t* pend;     // [LOGCAP] nodes whose slot word was not published yet
  int* nlog;          // [4] created, pending, dirty
  uint4* dbuf;        // [DBUF] (node, prompt, child, 0): shallow parents whose csum changed
                      // (hub refresh) and the child counted, flushed in batches
  uint32_t* pdl;      // null: flushed to the global dirty list; else the warp's prompt's own
                      // list ([0] count, then (hub, child) pairs: the fused tree step)
};
constexpr int DBUF = 96;

__host__ __device__ __forceinline__ size_t cursor_warp_bytes(int32_t D) {
  const size_t a = ((size_t)(D + 1) * 4 + 15) & ~size_t(15);
  const size_t f = ((size_t)(D + 1) + 15) & ~size_t(15);
  return a + f + (size_t)LOGCAP * 16 + 16 + (size_t)DBUF * 16;
}

// The dirty log (parents whose csum changed, for the hub refresh) is kept in
// shared memory and appended to the global list once per batch: a global
// append per position would put an atomic round trip on the insert's
// critical path.
__device__ __forceinline__ void dirty_flush(const DevCache& c, const CursorSmem& S, int lane) {
  __syncwarp();
  const int nd = S.nlog[2];
  if (nd) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(S.pdl ? S.pdl : c.dirty_n, (uint32_t)nd);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < nd; i += 32) {
      const uint4 e = S.dbuf[i];
      if (S.pdl) {
        if (base + i < PDIRTY_CAP) {
          S.pdl[2 + 2 * (base + i)] = e.x;
          S.pdl[3 + 2 * (base + i)] = e.z;
        }
      } else if (base + i < DIRTY_CAP) {
        c.dirty[base + i] = make_uint2(e.x, e.y);
      }
    }
  }
  __syncwarp();
  if (lane == 0) S.nlog[2] = 0;
  __syncwarp();
}
__device__ __forceinline__ void dirty_push(const DevCache& c, const CursorSmem& S, bool want,
                                           uint32_t u, int32_t p, uint32_t child, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  if (S.nlog[2] + __popc(m) > DBUF) dirty_flush(c, S, lane);
  const int nd = S.nlog[2];
  if (want) S.dbuf[nd + __popc(m & lanemask_lt())] = make_uint4(u, (uint32_t)p, child, 0u);
  __syncwarp();
  if (lane == 0) S.nlog[2] = nd + __popc(m);
  __syncwarp();
}

// Link the logged nodes, publish their slot words and add the mirror counts;
// then the mirror counts of the pending nodes (their creators publish in
// their own batches, which never wait on this warp's pending list).  Each lane
// takes FL entries at a time with their first round trips in flight together.
constexpr int FL = 8;
__device__ void cursor_flush(const DevCache& c, const CursorSmem& S, int lane) {
  __syncwarp();
  const int nc = S.nlog[0], np = S.nlog[1];
  for (int b = 0; b < nc; b += 32 * FL) {
    uint32_t k0[FL];
#pragma unroll
    for (int i = 0; i < FL; ++i) {  // claim the child index: all in flight
      const int e = b + i * 32 + lane;
      k0[i] = e < nc ? atomicAdd(&rec_of(c, S.log_par[e])->x, 1u) : 0u;
    }
#pragma unroll
    for (int i = 0; i < FL; ++i) {
      const int e = b + i * 32 + lane;
      if (e >= nc) continue;
      const uint32_t h = S.log_h[e], u = S.log_par[e];
      const int32_t tkf = S.log_tok[e];
      const bool counted = tkf >= 0;  // (walk hops before `from` create without counting)
      const int32_t tk = tkf & 0x7FFFFFFF;
      uint32_t pos;
      if (k0[i] == 0) {  // inline child 0 (read only by later kernels)
        uint4* r = rec_of(c, u);
        r->y = h;
        r->z = (uint32_t)tk;
        pos = AUX_CHILD0;
      } else {
        pos = place_child(c, u, k0[i] - 1, h, tk);
      }
      st_relaxed_u32(&c.hash[h].aux, pos);
      if (counted && is_slot_word(pos)) atomicAdd(&c.scnt[pos], 1u);
    }
  }
  __syncwarp();
  for (int b = 0; b < np; b += 32 * FL) {
    uint32_t a[FL];
#pragma unroll
    for (int i = 0; i < FL; ++i) {  // read the slot words: all in flight
      const int e = b + i * 32 + lane;
      a[i] = e < np ? ld_relaxed_u32(&c.hash[S.pend[e]].aux) : AUX_CHILD0;
    }
#pragma unroll
    for (int i = 0; i < FL; ++i) {
      const int e = b + i * 32 + lane;
      if (e >= np) continue;
      const uint32_t pos = a[i] != NONE ? a[i] : wait_aux(c, S.pend[e]);
      if (is_slot_word(pos)) atomicAdd(&c.scnt[pos], 1u);
    }
  }
  __syncwarp();
  if (lane == 0) S.nlog[0] = S.nlog[1] = 0;
  __syncwarp();
}

// This warp's slice of the cursor kernels' dynamic shared memory.
__device__ __forceinline__ CursorSmem carve_cursor_smem(unsigned char* base, int w, int32_t D) {
  CursorSmem S;
  unsigned char* b = base + (size_t)w * cursor_warp_bytes(D);
  S.A = reinterpret_cast<uint32_t*>(b);
  b += ((size_t)(D + 1) * 4 + 15) & ~size_t(15);
  S.fresh = b;
  b += ((size_t)(D + 1) + 15) & ~size_t(15);
  S.log_h = reinterpret_cast<uint32_t*>(b);
  S.log_par = S.log_h + LOGCAP;
  S.log_tok = reinterpret_cast<int32_t*>(S.log_par + LOGCAP);
  S.pend = reinterpret_cast<uint32_t*>(S.log_tok + LOGCAP);
  S.nlog = reinterpret_cast<int*>(S.pend + LOGCAP);
  S.dbuf = reinterpret_cast<uint4*>(S.nlog + 4);
  S.pdl = nullptr;
  return S;
}

// The cursor insertion of sequence s's span [f, t_end) by one warp (prompt p
// already checked).
template <int NG, bool MW = false>  // D <= 32 * NG; MW: NG warps per sequence, one group each
__device__ __forceinline__ void cursor_insert_seq(
    const DevCache& c, const CursorSmem& S, int32_t s, int32_t p, int32_t f, int32_t t_end,
    const int32_t* __restrict__ seq_tok, int64_t stride, const int32_t* __restrict__ floor_,
    int32_t short_max, uint32_t* __restrict__ cursor, uint32_t tag, srt_insert_stats* stats) {
  const int lane = threadIdx.x & 31;
  // MW: warp gw of the sequence's NG warps owns depth group gw (S.A is shared
  // by the warps; logs are per warp), synchronised once per position
  const int gw = MW ? (int)(threadIdx.x >> 5) : 0;
  constexpr int NGL = MW ? 1 : NG;  // depth groups per lane
  constexpr int LSTRIDE = MW ? 32 * NG : 32;
  const int32_t D = c.D;
  uint32_t* cur = cursor + (size_t)s * (D + 4);
  const int32_t fl = floor_ ? floor_[s] : 0;
  const int32_t P = max(f, fl);
  if (t_end <= P) return;  // no window ends at a new position: cursor untouched
  if (t_end - P > short_max) {  // long span: the walk kernel inserts it
    if (lane == 0) cur[1] = NONE;  // and the cursor must be rebuilt next time
    return;
  }
  long long* const prof = g_ins_prof;
  const long long tp0 = clock64();
  long long tp_cur = 0, tp_max = 0, tp_batch = 0, tp_res = 0, tp_cnt = 0, rounds = 0;
  const int32_t* y = seq_tok + (int64_t)s * stride;
  unsigned incs = 0, created = 0;
  const bool valid = cur[0] == tag && cur[1] == (uint32_t)P && cur[2] == (uint32_t)p &&
                     cur[3] == (uint32_t)fl;
  if (lane == 0) {
    S.A[0] = root_id(c, p);
    S.fresh[0] = 0;
    S.nlog[0] = S.nlog[1] = S.nlog[2] = 0;
  }
  if (valid) {
    for (int32_t l = 1 + 32 * gw + lane; l <= D; l += LSTRIDE) {
      S.A[l] = cur[4 + l - 1];
      S.fresh[l] = 0;
    }
  } else {
    // rebuild: A_l for l <= min(D-1, P-floor) by walking y[P-l .. P-1] from the
    // root (creating missing nodes, counting nothing: these windows end < P)
    const int32_t lmax = min(D - 1, P - max(fl, 0));
    for (int32_t l = 1 + 32 * gw + lane; l <= D; l += LSTRIDE) {
      uint32_t u = NONE;
      if (l <= lmax) {
        u = root_id(c, p);
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
      S.A[l] = u;
      S.fresh[l] = 0;
    }
  }
  if (MW) __syncthreads(); else __syncwarp();
  tp_cur = clock64() - tp0;
  constexpr int ngroups = NGL;
  int32_t ybuf = 0;  // the span's tokens, 32 positions per load (lane i: position j + i)
  for (int32_t j = P; j < t_end; ++j) {
    const long long tj = clock64();
    if (((j - P) & 31) == 0) ybuf = j + lane < t_end ? y[j + lane] : 0;
    const int32_t tk = __shfl_sync(0xffffffffu, ybuf, (j - P) & 31);
    const bool oov = tk < 0 || tk >= c.V;
    if (oov && lane == 0) set_error(c, SRT_DEV_OOV);
    const int32_t lim = min(D, j - max(fl, 0) + 1);  // windows ending at j start >= floor
    uint32_t par[NGL], hnew[NGL], aux[NGL];
    bool act[NGL], cre[NGL];
    unsigned long long key[NGL];
#pragma unroll
    for (int g = 0; g < NGL; ++g) {
      const int32_t l = 32 * (gw + g) + lane + 1;
      par[g] = l <= D ? S.A[l - 1] : NONE;
      act[g] = l <= D && !oov && l <= lim && par[g] < BAD;
      key[g] = act[g] ? edge_key(par[g], (uint32_t)tk) : 0ull;
    }
    const long long tr = clock64();
    rounds += probe_edges<NGL>(c, key, act, hnew, cre, aux);
    // counts (fire and forget) and the batch logs (warp-aggregated appends)
    const long long tc = clock64();
    tp_res += tc - tr;
#pragma unroll
    for (int g = 0; g < NGL; ++g) {
      if (g >= ngroups) break;  // (warp-uniform)
      const bool a = act[g];
      const uint32_t h = hnew[g];
      if (a) {
        atomicAdd(&c.cnt[h], 1u);
        atomicAdd(&rec_of(c, par[g])->w, 1u);
        ++incs;
        if (cre[g]) c.tok[h] = tk;
        else if (is_slot_word(aux[g])) atomicAdd(&c.scnt[aux[g]], 1u);
      }
      if (gw + g == 0) {  // shallow parents whose csum changed: their hub lists are rebuilt after the call
        const int32_t l = lane + 1;
        dirty_push(c, S, a && l >= 2 && l <= 1 + HUB_DIRTY_DEPTH, par[g], p, h, lane);
      }
      const unsigned mc = __ballot_sync(0xffffffffu, a && cre[g]);
      const unsigned mp = __ballot_sync(0xffffffffu, a && !cre[g] && aux[g] == NONE);
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
          S.log_par[e] = par[g];
          S.log_tok[e] = tk;
          ++created;
        }
        if (mp >> lane & 1) S.pend[bp + __popc(mp & lt)] = h;
      }
    }
    __syncwarp();
    tp_cnt += clock64() - tc;
    if (MW) __syncthreads();  // every warp has read its parents of this position
#pragma unroll
    for (int g = 0; g < NGL; ++g) {
      if (g >= ngroups) continue;
      const int32_t l = 32 * (gw + g) + lane + 1;
      if (l > D) continue;
      S.A[l] = act[g] ? hnew[g] : NONE;
      S.fresh[l] = act[g] && cre[g];
    }
    if (MW) __syncthreads(); else __syncwarp();
    tp_max = max(tp_max, clock64() - tj);
    // Mid-span flush when a log is nearly full.  MW: the decision is
    // block-wide, so every warp of the sequence publishes its created nodes
    // before any of them can spin in the pending loop on another CTA's node
    // (a per-warp decision could park a creator at the position barrier
    // while its sibling spins: a cross-CTA wait cycle).
    const bool over = S.nlog[0] > LOGCAP - 32 * MAXG || S.nlog[1] > LOGCAP - 32 * MAXG;
    if (MW ? __syncthreads_or(over) : over) cursor_flush(c, S, lane);
  }
  {
    const long long tb = clock64();
    cursor_flush(c, S, lane);
    dirty_flush(c, S, lane);
    tp_batch = clock64() - tb;
  }
  for (int32_t l = 1 + 32 * gw + lane; l <= D; l += LSTRIDE) cur[4 + l - 1] = S.A[l];
  if (lane == 0 && gw == 0) {
    cur[0] = tag;
    cur[1] = (uint32_t)t_end;
    cur[2] = (uint32_t)p;
    cur[3] = (uint32_t)fl;
  }
  count_created(c, created);
  if (prof) {
    unsigned long long d = created;
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0 && gw == 0) {  // (MW: warp 0's part)
      long long* o = prof + 8 * (int64_t)s;
      o[0] = clock64() - tp0;
      o[1] = tp_cur;
      o[2] = t_end - P;
      o[3] = (long long)d;
      o[4] = tp_max;
      o[5] = valid;
      o[6] = (tp_batch << 20) | rounds;
      o[7] = (tp_res << 32) | (tp_cnt & 0xFFFFFFFFll);
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
      if (gw == 0) atomicAdd(&stats->windows, (unsigned long long)(t_end - lo));
      atomicAdd(&stats->increments, b);
      if (d) atomicAdd(&stats->nodes_created, d);
    }
  }
}

}  // namespace
}  // namespace srt
