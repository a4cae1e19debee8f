// srt_internal.cuh — device-side data structures and primitives of libsrt.
//
// Layout of one cache in HBM.  All prompts share one node pool.
// A node's id IS the index of its edge's slot in the hash (so a lookup or a
// CAS that claims a new edge yields the child's id with no allocation step);
// the root of prompt p's tree T_p is node H + p.  Node arrays are
// sized H + P:
//   tok[]      i32  token labelling the edge into the node
//   cnt[]      u32  count(u) ("frequency statistics"; reading O1)
//   rec[]      32 B {nchild, child0, token of child0, csum, base of child
//                   blocks 0..3 (+1; 0 = not yet created)}: one load per pop;
//                   csum = sum of the children's counts (the denominator of
//                   C(v)), maintained by insert alongside cnt
//   hash[H]    16 B open-addressing edge hash: key (parent << 32) | token, the
//                   child's slot word in aux (the child's id = the slot index);
//                   keys (node << 32) | 0x80000000 | i -> word offset of child
//                   block i >= 4 in val (blocks 0..3 are in the record)
//   slots[W]   u32  child-id blocks for children 1.. : 4, 4, 8, 16, 32, 64, ...
//                   (geometric, so a hub node with F children has O(log F) blocks)
//   stok[W], scnt[W]  the token and a mirror of the count of the child in each
//                   slot, so a node's children enumerate with coalesced loads
// Concurrency: insertion creates nodes with a CAS on the hash key and publishes
// the child's slot word afterwards (polled by racing threads that need it);
// counts are atomic adds, so the logical tree
// (set of (path, count)) does not depend on scheduling.  Node ids do, but no
// output exposes them (draft order uses counts + tokens only; O8/O15).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/srt.h"

// Read-only loads of tree data.  A kernel that reads tree data other warps
// wrote in the SAME launch (the fused tree step, step.cu, defines
// SRT_COHERENT_LOADS before any include) must not use the non-coherent
// read-only path (ld.global.nc is outside the memory model): it uses
// ordinary loads, which the memory model orders after the acquire of the
// release that published the data (step.cu's per-prompt ready flags).
#ifdef SRT_COHERENT_LOADS
#define SRT_LDG(p) (*(p))
#define SRT_LD(x) (x)
#else
#define SRT_LDG(p) __ldg(p)
#define SRT_LD(x) (x)
#endif

namespace srt {

constexpr uint32_t NONE = 0xFFFFFFFFu;  // "no block" / "value pending"
constexpr uint32_t BAD = 0xFFFFFFFEu;   // creation failed (capacity): walk stops
constexpr uint32_t AUX_CHILD0 = 0xFFFFFFFDu;  // edge aux: the child is its parent's inline child 0
constexpr unsigned long long EMPTY_KEY = ~0ull;
// a removed edge or block key (srt_cache_prune): matches no key and is not
// EMPTY, so probe sequences through it stay intact; its slot is not reused
constexpr unsigned long long TOMB_KEY = ~0ull - 1;
constexpr uint32_t BLOCK_TAG = 0x80000000u;  // tokens are < 2^31

// Edge entries: aux = the child's slot word in its parent's child blocks
// (AUX_CHILD0 for the inline child 0; NONE until published), val unused.
// Block entries (blocks >= 4): val = the block's first slot word (NONE until
// published).
struct alignas(16) HashSlot {
  unsigned long long key;
  uint32_t val;
  uint32_t aux;
};

// Exact noise bounds: g over the 2^23 noise inputs, bucketed by
// r >> 13 (1024 buckets), plus the global max.
constexpr int NOISE_BUCKETS = 1024;
constexpr int NOISE_BUCKET_SHIFT = 13;

struct DevCache {
  int32_t V, P, D, L, Bmax, b0, snum, sden;
  double min_score;
  unsigned long long N, H, W;
  int32_t* tok;
  uint32_t* cnt;
  uint4* rec;  // 2 per node: [2u] = {nchild, child0, token of child0, csum},
               //             [2u+1] = child block bases 0..3, each + 1 (0 = none yet)
  HashSlot* hash;
  uint32_t* slots;  // child ids (children 1.. of a node, in its blocks)
  int32_t* stok;    // their tokens (immutable)
  uint32_t* scnt;   // mirrors of their counts, contiguous for enumeration
  unsigned long long* ctr;  // [0] nodes created (+ P roots), [1] next slot word
  uint32_t* status;         // sticky SRT_DEV_* bits
  uint32_t* sched;          // [2] the scan's row-claim counters (0 between launches)
  // the fused tree step (step.cu): per prompt, sequences in the batch, sequences
  // committed and inserted, list refresh done; drafts done; and each prompt's
  // dirty hubs ([0] count, then PDIRTY_CAP nodes; consumed by its refresh)
  uint32_t* st_pcount;      // [P]
  uint32_t* st_pdone;       // [P]
  uint32_t* st_pready;      // [P] 0 = inserting, 1 = hub refresh tasks published, 2 = ready
  uint32_t* st_pnd;         // [P] refresh tasks (the prompt's dirty hubs)
  uint32_t* st_pnext;       // [P] next task to claim
  uint32_t* st_pfin;        // [P] tasks finished
  uint32_t* st_ndone;       // [1]
  uint32_t* pdirty;         // [P][PDIRTY_WORDS]: [0] touches, then (hub, child) pairs, then
                            // the task starts (the pairs sorted by hub)
  float* gbound;  // [0, 1024) bucket maxima, [1024] global max, [1025, 2049) bucket minima of
                  // G64; [2049, 3073) bucket maxima of the single-word Gumbel g(r)
  // Hub child lists: for a node with more than HUB_MIN
  // children, its top HUB_K children by (count desc, token asc), valid while
  // the node's child count and csum are what they were when the list was
  // built (counts only grow: an unchanged csum means unchanged counts).
  // Direct-mapped by mix64(node) & (HC - 1); rebuilt after every insert for
  // the hubs the insert touched (the dirty list).
  uint32_t HC;
  uint32_t* hub_node;   // [HC] NONE = empty
  uint32_t* hub_nch;    // [HC]
  uint32_t* hub_csum;   // [HC]
  uint32_t* hub_len;    // [HC]
  uint32_t* hub_child;  // [HC][HUB_K] child ids, best first
  int32_t* hub_tok;     // [HC][HUB_K]
  uint32_t* hub_cnt;    // [HC][HUB_K]
  unsigned long long* hub_claim;  // [HC] (insert call << 32 | node) of the last refresh claim
  uint32_t hub_shift;   // log2 of the slots per prompt: prompt p's hubs live in slots
                        // [p << hub_shift, (p + 1) << hub_shift) (a refresh of one prompt never
                        // rewrites a list another prompt's draft may be reading)
  uint2* dirty;         // [DIRTY_CAP] (node, prompt): parents whose csum an insert changed (shallow ones) and hubs a draft found without a valid list
  uint32_t* dirty_n;    // [0] entries, [1] refresh generation (a device counter: graph-safe)
};

constexpr uint32_t HUB_MIN = 64;  // listed above this fan-out (measured: 32 / 128 / 256 slower or equal)
constexpr int HUB_K = 64;          // >= Bmax
constexpr uint32_t DIRTY_CAP = 1u << 20;
// fused tree step (step.cu): per prompt, the (hub, child) count increments of
// the step's inserts at shallow parents (child NONE: a hub a draft met
// without a valid list), then the refresh tasks (one per distinct hub)
constexpr uint32_t PDIRTY_CAP = 255;
// [0] count, [1] pad, pairs at 2 + 2i, task ranges (u32 pairs, 8-byte aligned) at 2 + 2 CAP
constexpr size_t PDIRTY_WORDS = 2 + 4 * (size_t)PDIRTY_CAP;
constexpr int HUB_DIRTY_DEPTH = 2;  // parents at depth 1..2 are logged as dirty

// Candidate (z, v) packed so that a larger u64 is the better candidate under
// "larger z, then smaller v" (first maximum): order-preserving float key in the
// high word (-0 folded onto +0, which compare equal), ~v in the low word.
// 0 is "no candidate".  z must not be NaN.
__device__ __forceinline__ unsigned long long pack_cand(float z, int32_t v) {
  uint32_t b = __float_as_uint(z == 0.0f ? 0.0f : z);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (0xFFFFFFFFu - (uint32_t)v);
}
__device__ __forceinline__ int32_t unpack_index(unsigned long long k) {
  return k ? (int32_t)(0xFFFFFFFFu - (uint32_t)k) : 0;
}
__device__ __forceinline__ float unpack_value(unsigned long long k) {
  const uint32_t b = (uint32_t)(k >> 32);
  return __uint_as_float((b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b);
}

// ---------------------------------------------------------------------------
// memory-model helpers (gpu scope; L1 is not coherent, so polled words use
// relaxed/acquire loads that go to L2)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Publish a hash slot's (val, aux) pair with one 64-bit store.  Relaxed is
// enough: within an insert kernel a waiter needs only these two words (the
// creator's other writes -- tok, child-0 fields, slot mirrors -- are read by
// later kernels only, and counts are atomics on zero-initialised memory), and
// kernel boundaries order everything for the readers.
__device__ __forceinline__ void publish_slot(HashSlot* s, uint32_t val, uint32_t aux) {
  const unsigned long long v = ((unsigned long long)aux << 32) | val;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&s->val), "l"(v) : "memory");
}

__device__ __forceinline__ void set_error(const DevCache& c, uint32_t bits) {
  atomicOr(c.status, bits);
}

// splitmix64 finaliser as the hash mixer
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Home slot of a key: linear probing from an EVEN slot, so the first two
// probes are one aligned 32-byte load (insert reads slot pairs).
__device__ __forceinline__ unsigned long long home_slot(const DevCache& c, unsigned long long key) {
  return mix64(key) & (c.H - 1) & ~1ull;
}

__device__ __forceinline__ unsigned long long edge_key(uint32_t parent, uint32_t tok) {
  return ((unsigned long long)parent << 32) | tok;
}
__device__ __forceinline__ unsigned long long block_key(uint32_t node, uint32_t i) {
  return ((unsigned long long)node << 32) | (BLOCK_TAG | i);
}

// ---- child-block geometry for children 1.. (slot j = child j+1):
//      blocks of 4, 4, 8, 16, 32, 64, ... slots (block i >= 2 holds [2^(i+1), 2^(i+2)))
__device__ __forceinline__ uint32_t blk_index(uint32_t j) {
  return j < 8 ? (j >> 2) : (uint32_t)(30 - __clz(j));
}
__device__ __forceinline__ uint32_t blk_start(uint32_t i) { return i < 2 ? 4u * i : (4u << (i - 1)); }
__device__ __forceinline__ uint32_t blk_size(uint32_t i) { return i < 2 ? 4u : (4u << (i - 1)); }

// Read-only lookup (kernels that run after all insertion is complete).
// Returns NONE if the key is absent.
__device__ __forceinline__ uint32_t hash_find(const DevCache& c, unsigned long long key) {
  unsigned long long mask = c.H - 1;
  unsigned long long h = home_slot(c, key);
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const HashSlot* s = c.hash + h;
    const unsigned long long k = SRT_LDG(&s->key);
    if (k == key) return SRT_LDG(&s->val);
    if (k == EMPTY_KEY) return NONE;
    h = (h + 1) & mask;
  }
  return NONE;
}

// Slot index of `key` (= the child's node id for an edge key), NONE if absent.
__device__ __forceinline__ uint32_t hash_slot(const DevCache& c, unsigned long long key) {
  unsigned long long mask = c.H - 1;
  unsigned long long h = home_slot(c, key);
  for (unsigned long long probe = 0; probe <= mask; ++probe) {
    const unsigned long long k = SRT_LDG(&c.hash[h].key);
    if (k == key) return (uint32_t)h;
    if (k == EMPTY_KEY) return NONE;
    h = (h + 1) & mask;
  }
  return NONE;
}

__device__ __forceinline__ uint32_t child_of(const DevCache& c, uint32_t u, int32_t tok) {
  return hash_slot(c, edge_key(u, (uint32_t)tok));
}

__device__ __forceinline__ uint32_t root_id(const DevCache& c, int32_t p) {
  return (uint32_t)(c.H + (unsigned long long)p);
}

// record of node u: {nchild, child0, token of child0, csum}
__device__ __forceinline__ uint4 ld_rec(const DevCache& c, uint32_t u) { return SRT_LDG(&c.rec[2 * (size_t)u]); }
__device__ __forceinline__ uint4* rec_of(const DevCache& c, uint32_t u) { return &c.rec[2 * (size_t)u]; }
// the record's block words (base of child block i < 4, + 1; 0 = not created)
__device__ __forceinline__ uint32_t* rec_bases(const DevCache& c, uint32_t u) {
  return reinterpret_cast<uint32_t*>(&c.rec[2 * (size_t)u + 1]);
}
// First slot word of child block i of node u (read-only kernels).
__device__ __forceinline__ uint32_t block_base(const DevCache& c, uint32_t u, uint32_t i) {
  if (i < 4) {
    const uint32_t b = SRT_LDG(rec_bases(c, u) + i);
    return b ? b - 1 : NONE;
  }
  return hash_find(c, block_key(u, i));
}

// Child k of node u (read-only kernels; slow path — enumeration loops look the
// block bases up once).  Child 0 is inline in rec; child k >= 1 is slot k-1.
__device__ __forceinline__ uint32_t child_at(const DevCache& c, uint32_t u, uint32_t child0,
                                             uint32_t k) {
  if (k == 0) return child0;
  const uint32_t j = k - 1;
  const uint32_t i = blk_index(j);
  return c.slots[block_base(c, u, i) + (j - blk_start(i))];
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Tree kernels may ask for the max-shared-memory L1 carveout, the one the
// verify scan runs with, so that their CTAs can co-reside with a running scan
// of another cache (env SRT_CARVEOUT=1; bench.py's pipelined schedule).
template <auto K>
inline void carveout_once() {
  static const bool done = [] {
    if (std::getenv("SRT_CARVEOUT"))
      cudaFuncSetAttribute((const void*)K, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)done;
}

// ---------------------------------------------------------------------------
// Launchers (defined in the .cu files; all enqueue on `stream`)
// ---------------------------------------------------------------------------
cudaError_t launch_init_cache(const DevCache& c, cudaStream_t stream);
cudaError_t launch_noise_bounds(const DevCache& c, cudaStream_t stream);
cudaError_t launch_noise_table(float* out, cudaStream_t stream);
cudaError_t launch_log_det_range(uint32_t first, int64_t n, float* out, cudaStream_t stream);
cudaError_t launch_row_noise(int32_t V, uint64_t seed, const uint64_t* seq_id, const int32_t* pos,
                             int32_t nkeys, float* out, cudaStream_t stream);
int num_sms();
cudaError_t launch_stream_read(const void* buf, int64_t bytes, int32_t chunk, int32_t nbuf,
                               int32_t ctas_per_sm, unsigned long long* sink, cudaStream_t stream);
cudaError_t launch_insert_plan(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* from, const int32_t* to, const int32_t* floor_,
                               int32_t short_max, long long* scratch, cudaStream_t stream);
cudaError_t launch_insert_cursor(const DevCache& c, int32_t n, const int32_t* prompt_id,
                                 const int32_t* seq_tok, int64_t stride, const int32_t* from,
                                 const int32_t* to, const int32_t* floor_, int32_t short_max,
                                 uint32_t* cursor, uint32_t tag, srt_insert_stats* stats,
                                 cudaStream_t stream);
size_t insert_cursor_smem(int32_t D);

cudaError_t launch_insert_walk(const DevCache& c, int32_t n, const int32_t* prompt_id,
                               const int32_t* seq_tok, int64_t stride, const int32_t* from,
                               const int32_t* to, const int32_t* floor_, srt_insert_stats* stats,
                               const long long* scratch, cudaStream_t stream);
cudaError_t launch_draft(const DevCache& c, int32_t n, const int32_t* prompt_id,
                         const int32_t* seq_tok, int64_t stride, const int32_t* seq_len,
                         const int32_t* pos_base, const uint32_t* cursor, uint32_t tag,
                         int32_t* match_len, int32_t* draft_len,
                         int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                         int32_t* draft_pos, uint64_t* draft_mask, cudaStream_t stream);
cudaError_t set_draft_profile(long long* buf);
cudaError_t set_insert_profile(long long* buf);
cudaError_t launch_row_offsets(int32_t n, const int32_t* draft_len, int64_t* row_offsets,
                               cudaStream_t stream);
struct VerifyArgs {
  int32_t n;
  const void* logits;
  int dtype;
  const int64_t* row_offsets;
  const int32_t* draft_len;
  const int32_t* draft_tok;
  const int32_t* draft_parent;
  const int32_t* draft_depth;
  const uint64_t* seq_id;
  uint64_t seed;
  float temperature;
  int32_t eos_id;
  const int32_t* max_new;
  int32_t* seq_tok;
  int64_t stride;
  int32_t* seq_len;
  int32_t* sampled;
  int32_t* accept_len;
  int32_t* n_commit;
  int32_t* commit_tok;
  int32_t* accepted_nodes;
  uint8_t* finished;
};
int scan_cluster_size(int32_t V, int dtype);
// per row: (sequence, position); clears result[row]
cudaError_t launch_rowinfo(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                           unsigned long long* result, cudaStream_t stream);
// the fused LM-head GEMM + Gumbel-max sampler (lmhead.cu): result[row] for
// every drafted row, logits never materialised (dump: optional debug copy)
struct LmHeadArgs {
  const void* hidden;   // bf16 [hidden_rows, K]
  int64_t hidden_rows;
  int32_t K;
  const void* weight;   // bf16 [V, K]
  void* dump;           // nullable: [rows, V] logits in cfg.logits_dtype
};
// per-row lists of the blocks the GEMM epilogue defers to the exact tail
struct LmHeadScratch {
  void* cand_x;     // [rows][cap][64] logits (cache dtype)
  int32_t* cand_b;  // [rows][cap]
  float* cand_X;    // [rows][cap]
  int32_t* cand_n;  // [rows], zero between calls
  int32_t cap;
};
constexpr int32_t LMHEAD_CAND_CAP = 256;
cudaError_t launch_lmhead_sample(const DevCache& c, const VerifyArgs& a, const LmHeadArgs& h,
                                 const int2* rowinfo, unsigned long long* result,
                                 const LmHeadScratch& sc, cudaStream_t stream);
cudaError_t launch_scan_cluster(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                                unsigned long long* result, cudaStream_t stream);
// reference = the unpruned kernel writing sampled[] directly; otherwise the
// product scan writing each row's packed winner (pack_cand) to result[].
cudaError_t launch_scan(const DevCache& c, const VerifyArgs& a, bool reference, int2* rowinfo,
                        unsigned long long* result, cudaStream_t stream);
cudaError_t launch_accept(const DevCache& c, const VerifyArgs& a, const unsigned long long* result,
                          cudaStream_t stream);
cudaError_t launch_tree_step(const DevCache& c, const VerifyArgs& a,
                             const unsigned long long* result, const int32_t* prompt_id,
                             const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                             srt_insert_stats* stats, const int32_t* pos_base, int32_t* match_len,
                             int32_t* draft_len, int32_t* draft_tok, int32_t* draft_parent,
                             int32_t* draft_depth, int32_t* draft_pos, uint64_t* draft_mask,
                             int64_t* row_offsets, cudaStream_t stream);
cudaError_t launch_accept_insert(const DevCache& c, const VerifyArgs& a,
                                 const unsigned long long* result, const int32_t* prompt_id,
                                 const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                                 srt_insert_stats* stats, cudaStream_t stream);
// seq_done (nullable): per-sequence count of rows whose result is final;
// grid_cap > 0: at most that many CTAs (the rest of the SMs run another kernel)
cudaError_t launch_scan_list(const DevCache& c, const VerifyArgs& a, const int2* rowinfo,
                             const int32_t* row_list, const int64_t* count,
                             unsigned long long* result, cudaStream_t stream,
                             uint32_t* seq_done = nullptr, int grid_cap = 0);
// the fused tree step beside the scan (step.cu): state words for n sequences
// of P prompts, its prep (before the scan), the per-sequence row counters the
// scan must count into, and the kernel (grid CTAs, each filling an SM)
size_t tree_step_ov_words(int32_t n, int32_t P);
cudaError_t launch_step_prep_ov(const DevCache& c, int32_t n, const int32_t* prompt_id,
                                const int64_t* row_offsets, uint32_t* ovbuf, cudaStream_t stream);
uint32_t* tree_step_ov_seq_done(uint32_t* ovbuf, int32_t n, int32_t P);
const int64_t* tree_step_ov_total(uint32_t* ovbuf, int32_t n, int32_t P);
cudaError_t launch_tree_step_ov(const DevCache& c, const VerifyArgs& a,
                                const unsigned long long* result, const int32_t* prompt_id,
                                const int32_t* floor_, uint32_t* cursor, uint32_t tag,
                                srt_insert_stats* stats, const int32_t* pos_base,
                                int32_t* match_len, int32_t* draft_len, int32_t* draft_tok,
                                int32_t* draft_parent, int32_t* draft_depth, int32_t* draft_pos,
                                uint64_t* draft_mask, int64_t* row_offsets, uint32_t* ovbuf,
                                int grid, cudaStream_t stream);
// path-only verification (srt_verify_path): scratch = 2 row lists + per-seq state
cudaError_t launch_path_verify(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                               unsigned long long* result, void* scratch, int rounds,
                               cudaStream_t stream);
size_t path_scratch_bytes(int32_t n, int32_t Bmax);
cudaError_t launch_pack_drafts(int32_t n, int32_t B, const int32_t* match_len,
                               const int32_t* draft_len, const int32_t* draft_tok,
                               const int32_t* draft_parent, const int32_t* draft_depth,
                               const uint64_t* draft_mask, int32_t* rec, cudaStream_t stream);
cudaError_t launch_unpack_drafts(int32_t n, int32_t B, const int32_t* rec, const int32_t* src,
                                 const int32_t* pos_base, int32_t* match_len, int32_t* draft_len,
                                 int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                                 int32_t* draft_pos, uint64_t* draft_mask, cudaStream_t stream);
cudaError_t launch_pack_spans(int32_t n, int32_t B, const int32_t* n_commit,
                              const int32_t* commit_tok, int32_t* rec, cudaStream_t stream);
cudaError_t launch_apply_spans(int32_t n, int32_t B, const int32_t* rec, const int32_t* src,
                               int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* from,
                               int32_t* to, cudaStream_t stream);
cudaError_t launch_prune_level(const DevCache& c, const uint32_t* front, int32_t nf, uint32_t theta,
                               uint32_t* next_keep, unsigned* n_keep, uint32_t* next_dead,
                               unsigned* n_dead, cudaStream_t stream);
cudaError_t launch_kill_level(const DevCache& c, const uint32_t* dead, int32_t nd,
                              uint32_t* next_dead, unsigned* n_dead, unsigned long long* removed,
                              cudaStream_t stream);
cudaError_t launch_count_hist(const DevCache& c, unsigned long long* hist, int32_t nb,
                              cudaStream_t stream);
cudaError_t launch_load_level(const DevCache& c, const uint32_t* parent_ids, const int32_t* par_idx,
                              const int32_t* tok, const unsigned long long* cnt, int32_t n,
                              uint32_t* out_ids, cudaStream_t stream);
cudaError_t launch_hub_refresh(const DevCache& c, uint32_t call, uint32_t* work, uint32_t* work_n,
                               cudaStream_t stream);
// the hub-list slot of node u of prompt p (direct-mapped inside p's partition)
__device__ __forceinline__ uint32_t hub_slot(const DevCache& c, int32_t p, uint32_t u) {
  return ((uint32_t)p << c.hub_shift) |
         (uint32_t)(mix64(0x4855420000000000ull ^ u) & ((1ull << c.hub_shift) - 1));
}
cudaError_t launch_dump_level(const DevCache& c, const uint32_t* frontier, int32_t nf,
                              uint32_t* out_node, int32_t* out_parent, int32_t* out_tok,
                              uint32_t* out_cnt, uint32_t* out_nchild, unsigned int* out_n,
                              cudaStream_t stream);

}  // namespace srt
