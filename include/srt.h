/*
 * srt.h — C ABI of the B200-native SRT hot path (libsrt.so).
 *
 * SRT = "Speculative Rollout with Tree-Structured Cache" (arXiv 2601.09083).
 * Citations: P:Lnn = line of PAPER.md (§3 "Method" unless noted); O1..O16 =
 * the readings listed in DESIGN.md where the paper is silent or ambiguous.
 *
 * One step of the path (reading O14):
 *     srt_draft   -> [policy forward on the drafted rows, outside this library]
 *     srt_verify  -> srt_insert
 * (srt_draft_cursor / srt_insert_cursor keep per-sequence suffix cursors;
 * srt_verify_insert_cursor is srt_verify + srt_insert_cursor in one call with
 * the accept walk and the insert fused.)
 *
 * Conventions common to every call
 * --------------------------------
 *  - Every array argument is a DEVICE pointer owned by the caller (e.g. a torch
 *    tensor's data_ptr()), in row-major layout, and must stay valid until the
 *    work enqueued on `stream` has completed.  The library owns only the cache
 *    pools, allocated in srt_cache_create and freed in srt_cache_destroy.
 *  - All work is enqueued on the caller's `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).  No call synchronises the stream,
 *    except srt_cache_dump and srt_cache_status, which are documented blocking.
 *    All calls on one cache must be ordered on one stream (no concurrent host
 *    calls on the same cache).  Every call is CUDA-graph capturable except
 *    srt_cache_create / destroy / dump / status.
 *  - Errors: every call returns an srt_status.  SRT_ERR_INVALID_* are detected
 *    on the host before anything is enqueued.  Problems only visible on the
 *    device (out-of-vocabulary token, exhausted pool, NaN logit, bad prompt id)
 *    set sticky bits in the cache's device status word, read by
 *    srt_cache_status.  SRT_DEV_CAPACITY poisons the cache: recreate it.
 *  - Sequence table: the caller's response tokens, seq_tok[s*stride + i] =
 *    response token i of sequence s (int32), seq_len[s] = tokens committed so
 *    far (t in the paper's y_{1:t}).  Prompt tokens are not part of it
 *    (reading O2/O3: windows and matches are response-only).
 *  - Token ids are int32 in [0, V).  Prompt ids are int32 in [0, P).
 *
 * Data layout in HBM (owned by the cache): a node pool shared by
 * all prompts (the root of prompt p's tree T_p, is node H + p) as
 * structure-of-arrays (token, count, and a 32-byte record {child count, first
 * child, its token, sum of the children's counts, bases of child blocks 0-3}),
 * an open-addressing edge hash ((parent << 32) | token; a node's id IS the
 * index of its edge's hash slot), and a pool of child slots in geometric
 * blocks (4, 4, 8, 16, 32, 64, ... slots) holding children 1.. with their
 * tokens and count mirrors for coalesced enumeration.
 */
#ifndef SRT_H_
#define SRT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRT_ABI_VERSION 1

#if defined(__GNUC__)
#define SRT_API __attribute__((visibility("default")))
#else
#define SRT_API
#endif

typedef enum {
  SRT_OK = 0,
  SRT_ERR_INVALID_CONFIG = 1, /* config violates a constraint below                   */
  SRT_ERR_INVALID_ARG = 2,    /* null pointer, negative size, bad handle, T <= 0      */
  SRT_ERR_CUDA = 3,           /* CUDA launch / allocation failure: srt_error_string() */
  SRT_ERR_DEVICE = 4          /* a sticky device error is set: see srt_cache_status   */
} srt_status;

/* Sticky device error bits (srt_cache_status). */
#define SRT_DEV_OOV 0x1u              /* a token >= V or < 0 was inserted/matched (window stops) */
#define SRT_DEV_CAPACITY 0x2u         /* node / hash / slot pool exhausted: cache is poisoned    */
#define SRT_DEV_BAD_PROMPT 0x4u       /* prompt id outside [0, P): the sequence is skipped       */
#define SRT_DEV_NONFINITE_LOGIT 0x8u  /* a NaN logit was read (NaN is never sampled, O11)        */
#define SRT_DEV_INCONSISTENT 0x10u    /* srt_cache_dump found a child-slot mirror (token/count)
                                         that disagrees with the node arrays: a library bug   */

typedef enum { SRT_BF16 = 0, SRT_F32 = 1 } srt_dtype;

typedef struct {
  int32_t vocab_size;       /* V >= 2                                                      */
  int32_t max_prompts;      /* P >= 1; prompt ids are dense in [0, P)                      */
  int32_t max_depth;        /* D >= 1: window depth, every substring of length <= D is     */
                            /*   indexed ("all substrings", reading O1/O2)           */
  int32_t max_match_len;    /* L, 1 <= L <= min(D, 32): suffix-match cap (O3)      */
  int32_t budget_max;       /* Bmax, 1 <= Bmax <= 64 (one u64 tree-mask word per node)     */
  int32_t budget_base;      /* B(q) = min(Bmax, b0 + floor(q*num/den))  (O5)       */
  int32_t budget_slope_num; /*   0 <= b0 <= Bmax, num >= 0, den >= 1                       */
  int32_t budget_slope_den;
  double min_path_score;    /* stop when the best frontier score is below this (O7); 0=off */
  int64_t node_capacity;    /* node pool size, >= P + 1                                    */
  int64_t hash_capacity;    /* edge-hash slots: a power of two >= 2*node_capacity          */
  int64_t slot_capacity;    /* child-block words (4 B each), >= node_capacity              */
  srt_dtype logits_dtype;   /* dtype of the logits passed to srt_verify                    */
} srt_config;

typedef struct srt_cache srt_cache; /* opaque */

/* Device-side counters accumulated by srt_insert (optional, device pointer). */
typedef struct {
  unsigned long long windows;       /* window starts walked               */
  unsigned long long increments;    /* count(u) += 1 operations (O1)      */
  unsigned long long nodes_created; /* nodes created by this call         */
} srt_insert_stats;

/* Host-side snapshot returned by srt_cache_status (blocking). */
typedef struct {
  uint64_t nodes_used;     /* including the P roots                 */
  uint64_t node_capacity;
  uint64_t slots_used;     /* child-block words                     */
  uint64_t slot_capacity;
  uint64_t hash_capacity;
} srt_cache_stats;

/* One record of the canonical dump (SPEC S:L148-149 format). */
typedef struct {
  int32_t token;      /* -1 for the root                                   */
  int32_t n_children;
  uint64_t count;     /* root: sum of its children's counts                */
} srt_dump_record;

SRT_API int srt_abi_version(void);
/* Human-readable text of the last SRT_ERR_CUDA on this host thread. */
SRT_API const char* srt_error_string(void);

/*
 * srt_cache_create — allocate and initialise the trees of P prompts in HBM
 * ("for each prompt p, a cache ... organized as a tree-structured cache
 * T_p"; held in HBM rather than CPU memory, BJ:north_star (1)).
 * Validates `cfg` (SRT_ERR_INVALID_CONFIG), allocates the pools with
 * cudaMallocAsync on `stream`, initialises them, and builds the exact Gumbel
 * noise bound tables used by srt_verify's pruning.  *out is set
 * on success only.  Blocking only for the host-side bookkeeping.
 */
SRT_API srt_status srt_cache_create(const srt_config* cfg, void* stream, srt_cache** out);

/* srt_cache_destroy — free the pools (stream-ordered).  NULL is a no-op. */
SRT_API srt_status srt_cache_destroy(srt_cache* cache, void* stream);

/*
 * srt_insert — batched insertion of decoded / run-ahead spans ("decoded
 * outputs of running rollouts are inserted online into T_p and node counts are
 * updated"; run-ahead tokens "are inserted into T_p"; reading O1).
 * For each span s < n: prompt prompt_id[s], tokens seq_tok[s*stride + i],
 * new positions [from[s], to[s]), first allowed window start floor_[s]
 * (floor_ may be NULL = 0).  Every window that ENDS at a new position gets +1:
 * for each end j in [max(from,floor), to) and each d in [1, min(D, j-floor+1)],
 * count(tokens[j-d+1 .. j]) += 1; missing nodes are created (lock-free CAS on
 * the edge hash; atomic counts, so the result is independent of scheduling).
 * stats_dev (device, nullable) is ACCUMULATED into.  n == 0 is a no-op.
 */
SRT_API srt_status srt_insert(srt_cache* cache, int32_t n, const int32_t* prompt_id,
                      const int32_t* seq_tok, int64_t stride, const int32_t* from,
                      const int32_t* to, const int32_t* floor_, srt_insert_stats* stats_dev,
                      void* stream);

/*
 * srt_insert_cursor — srt_insert with one suffix cursor per span: same
 * arguments and the SAME resulting tree (node set and counts), plus
 * `cursor`, a DEVICE array of n records of SRT_CURSOR_WORDS(D) uint32 words
 * owned by the caller (record s belongs to span s; keep a sequence at the same
 * index across calls).  A record remembers, for the position P it was left
 * at, the nodes of the suffixes y[P-l .. P-1] (l = 1..D), so the next call
 * reaches every window that ends at a new position with ONE hop from the
 * previous suffix node instead of a walk from the root (P:L151 online
 * insertion, done incrementally).  Record words: [0] cache tag, [1] P,
 * [2] prompt, [3] floor, [4 .. 4+D) suffix nodes.  A record is used only if
 * its tag is this cache's, P == max(from, floor) and prompt / floor match;
 * otherwise (e.g. zero-filled on first use) it is rebuilt from the root, so
 * any content is safe.  Spans with more than D new positions are inserted by
 * the walk path and leave their record invalid.  The record is updated to
 * P = to on return (unchanged if the span inserts nothing).
 */
#define SRT_CURSOR_WORDS(D) ((D) + 4)
/* The cursor calls (srt_insert_cursor, srt_verify_insert_cursor) need
 * cfg.max_depth <= SRT_CURSOR_MAX_DEPTH (SRT_ERR_INVALID_ARG otherwise,
 * returned before anything is enqueued); srt_insert has no such limit. */
#define SRT_CURSOR_MAX_DEPTH 128
SRT_API srt_status srt_insert_cursor(srt_cache* cache, int32_t n, const int32_t* prompt_id,
                             const int32_t* seq_tok, int64_t stride, const int32_t* from,
                             const int32_t* to, const int32_t* floor_, uint32_t* cursor,
                             srt_insert_stats* stats_dev, void* stream);

/*
 * srt_draft — batched longest-suffix match + best-first draft + tree layout
 * (P:L135-139).  For each sequence s < n (prompt prompt_id[s], response
 * seq_tok[s*stride ...] of length t = seq_len[s]):
 *  match   : q = largest q in [1, min(L, t)] such that the root walk along
 *            y[t-q .. t-1] exists and has >= 1 child (O3); q = 0 = fallback,
 *            empty draft ("revert to standard decoding for one step").
 *  expand  : C(v) = count(v) / sum of the counts of v and its siblings,
 *            score(v) = score(parent) * C(v), score(u_q) = 1 (fp64 RN, O6);
 *            pop the best frontier node under the total order O8 (score desc,
 *            depth asc, token asc, parent draft index asc) until B(q) nodes,
 *            an empty frontier, or best score < min_path_score.
 *  layout  : node i (pop order, 0 <= i < draft_len[s]) at [s*Bmax + i]:
 *            draft_tok, draft_parent (-1 = the root = last committed token),
 *            draft_depth (1 = child of the root), draft_pos = pos_base[s] + depth,
 *            draft_mask = ancestor-or-self bitmask over draft indices (bit i).
 *            Entries i >= draft_len[s] are tok=-1, parent=-1, depth=0, pos=-1,
 *            mask=0.  match_len[s] = q.  row_offsets[n+1] (int64) = exclusive
 *            scan of (draft_len + 1): the logits rows of sequence s are
 *            [row_offsets[s], row_offsets[s+1]) in the order [root, node 0, ...].
 * pos_base may be NULL (treated as 0).
 */
SRT_API srt_status srt_draft(srt_cache* cache, int32_t n, const int32_t* prompt_id,
                     const int32_t* seq_tok, int64_t stride, const int32_t* seq_len,
                     const int32_t* pos_base, int32_t* match_len, int32_t* draft_len,
                     int32_t* draft_tok, int32_t* draft_parent, int32_t* draft_depth,
                     int32_t* draft_pos, uint64_t* draft_mask, int64_t* row_offsets,
                     void* stream);

/*
 * srt_draft_cursor — srt_draft with the suffix cursors srt_insert_cursor
 * keeps (cursor[s*(D+4) ...], caller-owned DEVICE memory, read only).  Same
 * outputs as srt_draft.  When sequence s's cursor is valid for this cache and
 * sits at t = seq_len[s] with floor 0, its suffix nodes A_q are exactly the
 * nodes of y[t-q .. t-1], so the match (O3) reads the L candidates' records in
 * one round trip instead of walking q hops from the root; otherwise the
 * sequence walks as in srt_draft.
 */
SRT_API srt_status srt_draft_cursor(srt_cache* cache, int32_t n, const int32_t* prompt_id,
                                    const int32_t* seq_tok, int64_t stride, const int32_t* seq_len,
                                    const int32_t* pos_base, const uint32_t* cursor,
                                    int32_t* match_len, int32_t* draft_len, int32_t* draft_tok,
                                    int32_t* draft_parent, int32_t* draft_depth,
                                    int32_t* draft_pos, uint64_t* draft_mask,
                                    int64_t* row_offsets, void* stream);

/*
 * srt_verify — lossless verification ("verifies and accepts drafted
 * tokens up to the first mismatch"; "one decode pass ... verify
 * multiple drafted tokens in parallel"; readings O10, O11, O13).
 *  scan    : every logits row r of sequence s (row_offsets from srt_draft;
 *            logits has row_offsets[n] rows of V elements of cfg.logits_dtype)
 *            is sampled by Gumbel-max:  sampled[r] = argmax_v RN32(RN32(x_v/T)
 *            + g_v), smallest v on ties, NaN never chosen, where g_v is the
 *            block construction of reading O11: per block b of
 *            64 tokens (the last may be shorter, n_b), Philox4x32-10(ctr =
 *            (0x80000000 | b>>1, pos, seq_id lo, hi), key = (seed lo, hi))
 *            gives words (wa, wb) (words 0,1 for even b, 2,3 for odd b);
 *            E_b = RN(-log_det(u(wa)) / n_b), G_b = -log_det(E_b) is the
 *            block's maximum noise, at offset (wb * n_b) >> 32; every other
 *            v gets g_v = min(G_b, -log_det(RN(E_b + A_v))), A_v =
 *            -log_det(u(w_v)), w_v = word (v&3) of Philox4x32-10(ctr = (v>>2,
 *            pos, seq_id lo, hi)), u(w) = (2(w>>9)+1) 2^-24 -- i.e. n_b iid
 *            Gumbel(0,1) draws, the block maximum drawn first (top-down).
 *            pos = seq_len[s] for the root row, seq_len[s] + draft_depth for a
 *            node row.  T == 1 skips the division.  T must be > 0.
 *  walk    : from the root, accept the draft child whose token equals the
 *            current row's sample, until none does; accept_len[s] = a,
 *            accepted_nodes[s*Bmax + k] = draft index of the k-th accepted node
 *            (rest -1).
 *  commit  : the samples along the path (a accepted + 1 bonus token) are
 *            written to commit_tok[s*(Bmax+1) + k] (rest -1), truncated after
 *            the first eos_id (inclusive; eos_id < 0 = none) and at
 *            max_new[s] - seq_len[s]; n_commit[s] = tokens committed; they are
 *            appended to seq_tok (stride `stride`), seq_len[s] += n_commit[s],
 *            finished[s] = EOS committed || seq_len[s] >= max_new[s].
 * draft arrays are those srt_draft wrote (stride Bmax).  seq_tok must have
 * room for seq_len[s] + Bmax + 1 tokens per row.
 */
SRT_API srt_status srt_verify(srt_cache* cache, int32_t n, const void* logits,
                      const int64_t* row_offsets, const int32_t* draft_len,
                      const int32_t* draft_tok, const int32_t* draft_parent,
                      const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed,
                      float temperature, int32_t eos_id, const int32_t* max_new,
                      int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* sampled,
                      int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
                      int32_t* accepted_nodes, uint8_t* finished, void* stream);

/*
 * ---- Multi-GPU exchange records (BJ:north_star "prompts shard by hash across
 * the GPUs ... decoded spans are NCCL all-gathered over NVLink before
 * insertion").  A prompt's tree lives on its owner rank, which
 * keeps a mirror of its sequences' response tokens and drafts for them; the
 * drafts return to the decoding ranks and the committed spans go back to the
 * owners.  Records are fixed-size int32 rows so that one all-gather moves a
 * whole batch; these calls only pack, route and unpack them (stateless, no
 * cache needed).  All pointers are DEVICE pointers.
 *
 * Draft record (SRT_DRAFT_RECORD_WORDS(Bmax) words): [0] match_len, [1]
 * draft_len, then Bmax each of draft_tok, draft_parent, draft_depth, and the
 * low and high words of draft_mask.  (Positions are re-derived from the
 * receiving rank's pos_base.)
 * Span record (SRT_SPAN_RECORD_WORDS(Bmax) words): [0] n_commit, [1 ..]
 * commit_tok (Bmax + 1 words).
 */
#define SRT_DRAFT_RECORD_WORDS(Bmax) (2 + 5 * (Bmax))
#define SRT_SPAN_RECORD_WORDS(Bmax) ((Bmax) + 2)

/*
 * srt_verify_path — srt_verify that samples only the rows the commit needs
 * (SURVEY §8(f3b)).  The walk goes level by level: path_rounds rounds each
 * scan one row per sequence still accepting (its current node: the root,
 * then each accepted node), then every sequence still accepting has its
 * current node's whole draft subtree scanned at once and the walk finishes.
 * Same arguments and the same outputs as srt_verify -- commits, accept_len,
 * n_commit, commit_tok, accepted_nodes, finished, the sequence table, and
 * sampled[] for every row on the accepted path and the stopping row (the
 * same Gumbel-max draws, O11) -- except sampled[r] = -1 for rows not
 * sampled.  path_rounds = 0 samples every row (= srt_verify).  Requires
 * 16-byte-aligned rows (SRT_ERR_INVALID_ARG otherwise).  No host sync.
 */
SRT_API srt_status srt_verify_path(srt_cache* cache, int32_t n, int32_t path_rounds,
                                   const void* logits, const int64_t* row_offsets,
                                   const int32_t* draft_len, const int32_t* draft_tok,
                                   const int32_t* draft_parent, const int32_t* draft_depth,
                                   const uint64_t* seq_id, uint64_t seed, float temperature,
                                   int32_t eos_id, const int32_t* max_new, int32_t* seq_tok,
                                   int64_t stride, int32_t* seq_len, int32_t* sampled,
                                   int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
                                   int32_t* accepted_nodes, uint8_t* finished, void* stream);

/*
 * srt_verify_insert_cursor — srt_verify followed by srt_insert_cursor of the
 * committed spans, with the accept walk and the insert fused into one kernel
 * (per sequence, one warp -- D <= 32 -- or one CTA of ceil(D/32) warps, one
 * per depth group, commits its tokens, and inserts the windows ending
 * at them through its cursor right away, "updated online"; DESIGN.md
 * §5 f1).  Arguments: those of srt_verify, then prompt_id[n] (the tree each
 * sequence inserts into), floor[n] (nullable, as srt_insert), cursor[n][D + 4]
 * and stats (nullable), as srt_insert_cursor; the span of sequence s is
 * [seq_len_before, seq_len_after) -- every span goes through the cursor (at
 * most Bmax + 1 tokens, even when that exceeds D).  Results are identical to
 * srt_verify then srt_insert_cursor(from = the old seq_len, to = the new
 * one): the same outputs, trees and hub-list refresh, and cursor records for
 * the same suffixes
 * except for a span longer than D, after which srt_insert_cursor (walk path)
 * leaves the record invalid while this call keeps it valid at the new length.
 * D <= SRT_CURSOR_MAX_DEPTH.  Errors as both calls.
 */
SRT_API srt_status srt_verify_insert_cursor(
    srt_cache* cache, int32_t n, const void* logits, const int64_t* row_offsets,
    const int32_t* draft_len, const int32_t* draft_tok, const int32_t* draft_parent,
    const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed, float temperature,
    int32_t eos_id, const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len,
    int32_t* sampled, int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
    int32_t* accepted_nodes, uint8_t* finished, const int32_t* prompt_id, const int32_t* floor,
    uint32_t* cursor, srt_insert_stats* stats, void* stream);

/*
 * srt_verify_lmhead — srt_verify without materialised logits (
 * P:L139 "one decode pass", P:L379 decoding is memory-bandwidth bound): the
 * logits row r is the LM-head product x_r = hidden[r] . weight^T, computed on
 * the tensor cores (tcgen05, fp32 accumulation) and rounded to
 * cfg.logits_dtype (bf16: round-to-nearest-even, as a bf16 LM head stores
 * it); the sampler of srt_verify (reading O11: the same Gumbel-max, keys,
 * temperature and tie rule) runs as the GEMM's epilogue on those values, so
 * the [rows, V] logits never reach HBM.  Outputs and their meaning are
 * exactly srt_verify's run on the rounded logits.
 *   hidden      DEVICE bf16 [hidden_rows, hidden_dim], row r = the final
 *               hidden state of logits row r (rows as srt_draft lays them
 *               out: row_offsets[n] <= hidden_rows), 16-byte aligned;
 *   weight      DEVICE bf16 [V, hidden_dim] (the LM head / tied embedding),
 *               16-byte aligned; hidden_dim a multiple of 8;
 *   logits_out  nullable DEVICE [row_offsets[n], V] of cfg.logits_dtype: if
 *               given, the rounded logits the sampler saw are also written
 *               (test / debug support; it costs the write the fusion saves).
 * The accumulation order of the tensor-core GEMM is the hardware's, so the
 * logits themselves match an fp32 reference only to a tolerance; the
 * sampling is bit-exact given them.  SRT_ERR_INVALID_ARG for a bad shape or
 * alignment, SRT_ERR_CUDA if the tensor maps cannot be built.
 */
SRT_API srt_status srt_verify_lmhead(srt_cache* cache, int32_t n, const void* hidden,
                                     int64_t hidden_rows, int32_t hidden_dim, const void* weight,
                                     void* logits_out, const int64_t* row_offsets,
                                     const int32_t* draft_len, const int32_t* draft_tok,
                                     const int32_t* draft_parent, const int32_t* draft_depth,
                                     const uint64_t* seq_id, uint64_t seed, float temperature,
                                     int32_t eos_id, const int32_t* max_new, int32_t* seq_tok,
                                     int64_t stride, int32_t* seq_len, int32_t* sampled,
                                     int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
                                     int32_t* accepted_nodes, uint8_t* finished, void* stream);

/* srt_verify_lmhead + the fused accept and cursor insert of
 * srt_verify_insert_cursor (same extra arguments, same results). */
SRT_API srt_status srt_verify_lmhead_insert_cursor(
    srt_cache* cache, int32_t n, const void* hidden, int64_t hidden_rows, int32_t hidden_dim,
    const void* weight, void* logits_out, const int64_t* row_offsets, const int32_t* draft_len,
    const int32_t* draft_tok, const int32_t* draft_parent, const int32_t* draft_depth,
    const uint64_t* seq_id, uint64_t seed, float temperature, int32_t eos_id,
    const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len, int32_t* sampled,
    int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok, int32_t* accepted_nodes,
    uint8_t* finished, const int32_t* prompt_id, const int32_t* floor, uint32_t* cursor,
    srt_insert_stats* stats, void* stream);

/*
 * srt_verify_insert_draft_cursor — one call for everything after the policy
 * forward of step k: srt_verify_insert_cursor (the scan of every drafted row,
 * the commit, and the cursor insertion of the committed spans)
 * followed by srt_draft_cursor of step k + 1 over the updated
 * sequences, with the commit, insertion, hub-list refresh and next draft in
 * ONE persistent kernel ordered per prompt:
 * reading O14 orders draft(k+1) of prompt p after the inserts of p only, so
 * a prompt drafts as soon as its own sequences are committed and inserted.
 * Arguments: those of srt_verify_insert_cursor, then pos_base[n] (nullable;
 * read after the commit, so it may alias seq_len: positions = the new length
 * + depth) and the draft outputs of srt_draft (match_len ... row_offsets).
 * The draft outputs MAY alias this call's draft inputs (the same buffers):
 * sequence s's new draft is written only after its prompt's commits, and
 * row_offsets[0 .. n] only after every commit.  Results are identical to
 * srt_verify_insert_cursor then srt_draft_cursor(prompt_id, seq_tok,
 * seq_len, pos_base, cursor).  cfg.max_depth <= SRT_CURSOR_MAX_DEPTH (one
 * warp per sequence's insert for D <= 32, one CTA of ceil(D/32) warps above;
 * SRT_ERR_INVALID_ARG otherwise, before anything is enqueued).  The kernel
 * keeps every CTA resident (cross-warp waits): do not run another kernel
 * that could hold SMs indefinitely concurrently.  Device-side errors as both
 * calls.
 */
SRT_API srt_status srt_verify_insert_draft_cursor(
    srt_cache* cache, int32_t n, const void* logits, const int64_t* row_offsets,
    const int32_t* draft_len, const int32_t* draft_tok, const int32_t* draft_parent,
    const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed, float temperature,
    int32_t eos_id, const int32_t* max_new, int32_t* seq_tok, int64_t stride, int32_t* seq_len,
    int32_t* sampled, int32_t* accept_len, int32_t* n_commit, int32_t* commit_tok,
    int32_t* accepted_nodes, uint8_t* finished, const int32_t* prompt_id, const int32_t* floor,
    uint32_t* cursor, srt_insert_stats* stats, const int32_t* pos_base, int32_t* next_match_len,
    int32_t* next_draft_len, int32_t* next_draft_tok, int32_t* next_draft_parent,
    int32_t* next_draft_depth, int32_t* next_draft_pos, uint64_t* next_draft_mask,
    int64_t* next_row_offsets, void* stream);

/*
 * srt_cache_set_step_overlap — where srt_verify_insert_draft_cursor runs its
 * fused tree step.  sms > 0: on `sms` SMs BESIDE the scan,
 * which then runs on the other SMs: the step kernel is a programmatic
 * dependent launch on the caller's stream (it starts while the scan runs)
 * and commits and inserts each sequence as soon as the scan has finished
 * that sequence's rows, so the latency-bound tree work hides under the
 * HBM-bound scan.  If the two kernels do not overlap (a tool or another
 * context holding the SMs) the step kernel simply runs after the scan: the
 * scan never waits on it.  0: after the scan, on every SM.  -1: the library
 * default (SRT_STEP_OVERLAP in the environment overrides it).  Applies to
 * cfg.max_depth <= 32 and 16-byte aligned logits rows; other calls run the
 * step after the scan.  Results are identical in every mode.
 * SRT_ERR_INVALID_ARG unless -1 <= sms < the SM count.
 */
SRT_API srt_status srt_cache_set_step_overlap(srt_cache* cache, int32_t sms);

/* records[s] <- the draft of sequence s < n (srt_draft's outputs). */
SRT_API srt_status srt_pack_drafts(int32_t n, int32_t Bmax, const int32_t* match_len,
                           const int32_t* draft_len, const int32_t* draft_tok,
                           const int32_t* draft_parent, const int32_t* draft_depth,
                           const uint64_t* draft_mask, int32_t* records, void* stream);

/*
 * For s < n: unpack records[src[s]] into sequence s's draft outputs, with
 * draft_pos = pos_base[s] + depth (pos_base may be NULL = 0), padding as
 * srt_draft, and row_offsets[n+1] = exclusive scan of (draft_len + 1) -- the
 * same outputs srt_draft would have written for these sequences.
 */
SRT_API srt_status srt_unpack_drafts(int32_t n, int32_t Bmax, const int32_t* records,
                             const int32_t* src, const int32_t* pos_base, int32_t* match_len,
                             int32_t* draft_len, int32_t* draft_tok, int32_t* draft_parent,
                             int32_t* draft_depth, int32_t* draft_pos, uint64_t* draft_mask,
                             int64_t* row_offsets, void* stream);

/* records[s] <- {n_commit[s], commit_tok[s][0 .. Bmax]} (srt_verify's outputs). */
SRT_API srt_status srt_pack_spans(int32_t n, int32_t Bmax, const int32_t* n_commit,
                          const int32_t* commit_tok, int32_t* records, void* stream);

/*
 * Owner side: for mirror sequence m < n, append the k = records[src[m]][0]
 * committed tokens to its row of the mirror table (seq_tok[m*stride ...],
 * seq_len[m] += k, never past stride) and write the insertion span
 * from[m] = old length, to[m] = new length for srt_insert / srt_insert_cursor.
 */
SRT_API srt_status srt_apply_spans(int32_t n, int32_t Bmax, const int32_t* records,
                           const int32_t* src, int32_t* seq_tok, int64_t stride,
                           int32_t* seq_len, int32_t* from, int32_t* to, void* stream);

/*
 * srt_cache_dump — canonical serialization of T_p (BLOCKING; test path).
 * Preorder records, children in ascending token order.
 * host_buf (HOST pointer, capacity cap records) may be NULL to query the size;
 * *n_records receives the total record count.  Returns SRT_ERR_DEVICE if the
 * cache is poisoned.
 */
SRT_API srt_status srt_cache_dump(srt_cache* cache, int32_t prompt_id, srt_dump_record* host_buf,
                          int64_t cap, int64_t* n_records, void* stream);

/*
 * srt_cache_status — BLOCKING: synchronises `stream`, returns the sticky
 * device error bits (SRT_DEV_*) in *dev_error_bits and fills *stats (HOST
 * pointers; either may be NULL).  Returns SRT_ERR_DEVICE iff any bit is set.
 */
SRT_API srt_status srt_cache_status(srt_cache* cache, uint32_t* dev_error_bits, srt_cache_stats* stats,
                            void* stream);

/*
 * Capacity management and persistence (O17).  The
 * paper bounds nothing; these are maintenance calls between steps,
 * all BLOCKING (they synchronise `stream`), none on the per-step path.
 *
 * srt_cache_prune — remove every non-root node of T_p (every prompt if
 *   prompt_id = -1) whose count is below theta, i.e. the lowest-count whole
 *   subtrees (count(u) >= the count of each child, O1).  theta = UINT32_MAX
 *   resets T_p.  Kept children are compacted in their parents' child lists;
 *   removed edges become hash tombstones (their slots are not reused until the
 *   cache is rebuilt, e.g. by dump + load into a new cache).  Every insert
 *   cursor of this cache becomes invalid (rebuilt on its next use).
 *   *removed (HOST, nullable) = nodes removed.
 * srt_cache_evict — if more than max_nodes nodes are live, prune every tree
 *   with the smallest theta that leaves at most 0.9 * max_nodes (hysteresis,
 *   S:L121); *theta_out (HOST, nullable) = the theta used (0 = nothing done).
 * srt_cache_load — merge a canonical dump of T_p (srt_cache_dump's records,
 *   HOST memory) into T_p: paths are created as needed and counts added, so a
 *   dump loaded into an empty tree (a new cache, or after a reset) restores
 *   it exactly.  SRT_ERR_INVALID_ARG for a malformed list.
 */
SRT_API srt_status srt_cache_prune(srt_cache* cache, int32_t prompt_id, uint32_t theta,
                                   int64_t* removed, void* stream);
SRT_API srt_status srt_cache_evict(srt_cache* cache, int64_t max_nodes, int64_t* removed,
                                   uint32_t* theta_out, void* stream);
SRT_API srt_status srt_cache_load(srt_cache* cache, int32_t prompt_id,
                                  const srt_dump_record* host_buf, int64_t n_records, void* stream);

/* Clear the sticky error bits (not SRT_DEV_CAPACITY, which poisons). */
SRT_API srt_status srt_cache_clear_errors(srt_cache* cache, void* stream);

/*
 * srt_noise_table — test support: out[r] = g(r) = -log_det(-log_det((2r+1) 2^-24))
 * for all r in [0, 2^23) (DEVICE pointer, 2^23 floats): the plain per-word
 * Gumbel transform of O12 (the scan's noise is the block construction below,
 * srt_row_noise; this table is the bucket bound input of the block maxima).
 */
SRT_API srt_status srt_noise_table(float* out, void* stream);

/*
 * srt_log_det_range — test support: out[i] = log_det(x_i) for the n floats
 * whose bit patterns are first_bits, first_bits + 1, ... (DEVICE out, n
 * floats), with the device log_det every noise value goes through (reading
 * O12).  Lets a test compare log_det with the oracle's over
 * every positive normal float.  SRT_ERR_INVALID_ARG if the range passes 2^32.
 */
SRT_API srt_status srt_log_det_range(uint32_t first_bits, int64_t n, float* out, void* stream);

/*
 * srt_row_noise — test support: the sampler's noise g_v for every token v of
 * n row keys (reading O11, the top-down block construction): out[k*V + v] =
 * g_v for key (seed, seq_id[k], pos[k]) (DEVICE pointers; out has n*V
 * floats), computed by the device functions srt_verify's scan evaluates.
 * Lets a test compare every element's noise with the oracle bit for bit.
 */
SRT_API srt_status srt_row_noise(int32_t vocab_size, uint64_t seed, int32_t n,
                                 const uint64_t* seq_id, const int32_t* pos, float* out,
                                 void* stream);

/*
 * srt_stream_read — measurement support (not on the path): read the first
 * floor(bytes / chunk) * chunk bytes of the DEVICE buffer `buf` once through
 * shared memory (persistent kernel, ctas_per_sm CTAs per SM, nbuf stages of
 * chunk bytes, 1-D TMA bulk copies; SRT_STREAM_HINT=1 adds an L2 evict_first policy) and discard them; sink
 * is a DEVICE word it may write.  Timed by the caller with CUDA events, it is
 * the read-only HBM stream the verify scan is compared with.
 * SRT_ERR_INVALID_ARG unless chunk is a multiple of 1 KB and the stages fit
 * in 227 KB of shared memory per SM.
 */
SRT_API srt_status srt_stream_read(const void* buf, int64_t bytes, int32_t chunk, int32_t nbuf,
                                   int32_t ctas_per_sm, void* sink, void* stream);

/*
 * srt_sample_rows_reference — test support: the UNPRUNED scan (every element's
 * Philox + noise evaluated, one CTA per row) over the same rows as srt_verify's
 * scan stage; writes sampled[].  Used to show the pruned scan changes no bit.
 */
SRT_API srt_status srt_sample_rows_reference(srt_cache* cache, int32_t n, const void* logits,
                                     const int64_t* row_offsets, const int32_t* draft_depth,
                                     const int32_t* seq_len, const uint64_t* seq_id,
                                     uint64_t seed, float temperature, int32_t* sampled,
                                     void* stream);

/*
 * Per-kernel device timing (measurement support).  When enabled, every kernel
 * launched by srt_insert / srt_draft / srt_verify is bracketed by a pair of
 * CUDA events recorded on the caller's stream (up to `capacity` launches;
 * capacity 0 disables).  srt_profile_read (BLOCKING) synchronises `stream`,
 * returns the (kernel id, milliseconds) records in launch order into host_buf
 * (HOST, capacity cap) and clears them.
 */
typedef enum {
  SRT_K_INSERT_PLAN = 0,
  SRT_K_INSERT_WALK = 1,
  SRT_K_DRAFT = 2,
  SRT_K_ROW_OFFSETS = 3,
  SRT_K_SCAN = 4,
  SRT_K_ACCEPT = 5,
  SRT_K_INSERT_CURSOR = 6,
  SRT_K_HUB_REFRESH = 7, /* the hub child lists an insert call rebuilds */
  SRT_K_ACCEPT_INSERT = 8, /* srt_verify_insert_cursor's fused accept + cursor insert */
  SRT_K_LMHEAD = 9,        /* srt_verify_lmhead*: row info + the fused LM-head GEMM + sampler */
  SRT_K_TREE_STEP = 10     /* srt_verify_insert_draft_cursor: commit + insert + refresh + next draft */
} srt_kernel_id;

typedef struct {
  int32_t kernel; /* srt_kernel_id */
  float ms;
} srt_profile_record;

SRT_API srt_status srt_profile_enable(srt_cache* cache, int64_t capacity);
SRT_API srt_status srt_profile_read(srt_cache* cache, srt_profile_record* host_buf, int64_t cap,
                                    int64_t* n_records, void* stream);
/* As srt_profile_read but keeps the records: for launches captured in a CUDA
 * graph, each replay re-records the same event pairs, so peeking after a
 * replay (BLOCKING) returns that replay's per-kernel times. */
SRT_API srt_status srt_profile_peek(srt_cache* cache, srt_profile_record* host_buf, int64_t cap,
                                    int64_t* n_records, void* stream);

/*
 * srt_debug_draft_profile — development support: when dev_buf (DEVICE,
 * 8 int64 per sequence of the next srt_draft calls) is non-NULL, srt_draft
 * writes per sequence {cycles spent in the match, total cycles, children
 * enumerated, max children of one expanded node, cycles in record loads,
 * block lookups, child loads, frontier inserts}.  NULL disables (default).
 * Process-wide; not for concurrent use.
 */
SRT_API srt_status srt_debug_draft_profile(int64_t* dev_buf);

/*
 * srt_debug_insert_profile — development support: when dev_buf (DEVICE,
 * 8 int64 per sequence of the next srt_insert_cursor calls) is non-NULL, the
 * cursor kernel writes per sequence {total cycles, cycles loading or
 * rebuilding the cursor, new positions, nodes created, cycles of the slowest
 * position, cursor valid, 0, 0}.  NULL disables (default).  Process-wide.
 */
SRT_API srt_status srt_debug_insert_profile(int64_t* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* SRT_H_ */
