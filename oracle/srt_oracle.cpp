// =============================================================================
// SRT ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the per-step hot path
// of "Speculative Rollout with Tree-Structured Cache" (SRT, arXiv 2601.09083):
// insert -> longest-suffix match -> best-first draft -> Gumbel-max sample at
// every draft row -> first-mismatch walk + commit.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// leg may load this library. The product path (paper_2601_09083_b200/) never
// imports, links or executes it, and this file shares no code, header, table or
// constant generator with the CUDA path: every formula below is restated from
// the paper (PAPER.md, "P:Lnn") and from the readings in DESIGN.md ("O1".."O16").
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
// (no contraction / no fast-math: every float/double op below is one IEEE op).
//
// Parity status: every function here is pinned by a `-m "not gpu"` test
// (tests/test_oracle_*.py) against something other than itself — the paper's
// Fig. 3 worked example, brute-force enumeration, published Philox KATs, fp64
// libm accuracy bounds, closed-form invariants, and the losslessness property.
// =============================================================================
#include <cstdint>
#include <cstring>
#include <cmath>
#include <map>
#include <memory>
#include <queue>
#include <vector>
#include <algorithm>

namespace {

// ---------------------------------------------------------------------------
// Config (mirrors the fields DESIGN.md lists; plain struct, no shared header)
// ---------------------------------------------------------------------------
struct Config {
  int32_t vocab_size;        // V
  int32_t max_prompts;       // P
  int32_t max_depth;         // D: window depth (O2)
  int32_t max_match_len;     // L: suffix search cap (O3)
  int32_t budget_max;        // Bmax (<= 64)
  int32_t budget_base;       // b0
  int32_t budget_slope_num;  // B(q) = min(Bmax, b0 + floor(q*num/den))   (O5)
  int32_t budget_slope_den;
  double min_path_score;     // O7 (0 = off)
};

// ---------------------------------------------------------------------------
// Tree T_p: a node is a context, with out-edges labelled by the next
// token and a frequency count(u).  Children are kept in a std::map so they are
// always enumerated in ascending token order (canonical dump).
// ---------------------------------------------------------------------------
struct Node {
  int32_t tok = -1;
  uint64_t count = 0;
  std::map<int32_t, std::unique_ptr<Node>> kids;
};

struct Cache {
  Config cfg;
  std::vector<std::unique_ptr<Node>> roots;  // one root per prompt p
  uint32_t error_bits = 0;                   // 1 = OOV token, 4 = bad prompt id
  uint64_t nodes = 0;                        // non-root nodes created
};

Node* find_child(Node* u, int32_t tok) {
  auto it = u->kids.find(tok);
  return it == u->kids.end() ? nullptr : it->second.get();
}

Node* child_or_create(Cache* c, Node* u, int32_t tok) {
  auto it = u->kids.find(tok);
  if (it != u->kids.end()) return it->second.get();
  auto n = std::make_unique<Node>();
  n->tok = tok;
  Node* raw = n.get();
  u->kids.emplace(tok, std::move(n));
  c->nodes += 1;
  return raw;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11; the cuRAND/Random123 constants).
// Round: (hi0,lo0)=mulhilo(0xD2511F53,c0); (hi1,lo1)=mulhilo(0xCD9E8D57,c2);
//        c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key += (0x9E3779B9,0xBB67AE85)
// between rounds.  Pinned by the published KAT vectors (tests).
// ---------------------------------------------------------------------------
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

float f32_from_bits(uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; }
uint32_t bits_from_f32(float f) { uint32_t b; std::memcpy(&b, &f, 4); return b; }

// ---------------------------------------------------------------------------
// log_det (reading O12): a deterministic fp32 natural log built only from
// correctly-rounded IEEE operations, for positive normal x:
//   x = m * 2^e with m in [sqrt(1/2), sqrt(2)];  f = m - 1  (exact, Sterbenz)
//   s = f / (2 + f);  log(m) = 2 atanh(s) = 2s + s^3 (2/3 + 2/5 s^2 + ... )
//   log(x) = e*ln2 + log(m),  ln2 split into hi + lo parts.
// ---------------------------------------------------------------------------
float log_det(float x) {
  const float C3 = f32_from_bits(0x3f2aaaabu);   // RN32(2/3)
  const float C5 = f32_from_bits(0x3ecccccdu);   // RN32(2/5)
  const float C7 = f32_from_bits(0x3e924925u);   // RN32(2/7)
  const float C9 = f32_from_bits(0x3e638e39u);   // RN32(2/9)
  const float C11 = f32_from_bits(0x3e3a2e8cu);  // RN32(2/11)
  const float LN2_HI = f32_from_bits(0x3f317200u);
  const float LN2_LO = f32_from_bits(0x35bfbe8eu);
  uint32_t b = bits_from_f32(x);
  int32_t e = (int32_t)((b >> 23) & 0xFFu) - 127;
  uint32_t mb = (b & 0x007FFFFFu) | 0x3F800000u;
  if (mb > 0x3FB504F3u) {  // m > sqrt(2): halve m, bump e
    mb -= 0x00800000u;
    e += 1;
  }
  float m = f32_from_bits(mb);
  float f = m - 1.0f;
  float den = 2.0f + f;
  float s = f / den;
  float z = s * s;
  float p = std::fmaf(z, C11, C9);
  p = std::fmaf(z, p, C7);
  p = std::fmaf(z, p, C5);
  p = std::fmaf(z, p, C3);
  float sz = s * z;
  float two_s = 2.0f * s;
  float r = std::fmaf(sz, p, two_s);
  float ef = (float)e;
  float lo = std::fmaf(ef, LN2_LO, r);
  return std::fmaf(ef, LN2_HI, lo);
}

// Gumbel noise from one Philox word (reading O11):
//   r = w >> 9 (23 bits);  u = (2r+1) * 2^-24 in [2^-24, 1-2^-24] (exact in f32)
//   g = -log_det(-log_det(u))
float gumbel_from_word(uint32_t w) {
  uint32_t r = w >> 9;
  float u = (float)(2u * r + 1u) * f32_from_bits(0x33800000u);  // * 2^-24
  float a = -log_det(u);
  return -log_det(a);
}

float load_logit(const void* logits, int dtype, int64_t idx) {
  if (dtype == 0) {  // bf16: the high 16 bits of an f32
    uint16_t h = ((const uint16_t*)logits)[idx];
    return f32_from_bits((uint32_t)h << 16);
  }
  return ((const float*)logits)[idx];
}

// u(w) = (2 (w >> 9) + 1) 2^-24, exact in f32, in [2^-24, 1 - 2^-24]
float uniform_from_word(uint32_t w) {
  return (float)(2u * (w >> 9) + 1u) * f32_from_bits(0x33800000u);
}

// The Gumbel noise g_v of every element of one row (reading O11: the
// top-down construction of iid Gumbel variables, Maddison, Tarlow & Minka,
// "A* Sampling", NeurIPS 2014, §3 "Gumbel processes").  The vocabulary is cut
// into blocks of BLK = 64 consecutive tokens (the last may be shorter, n_b).
// For block b, one Philox4x32-10 call with counter (0x80000000 | (b >> 1),
// pos, seq_lo, seq_hi) gives two words (wa, wb) = words (0,1) for even b,
// (2,3) for odd b:
//   a_b  = -log_det(u(wa))              ~ Exp(1)
//   E_b  = RN(a_b / n_b)                ~ Exp(n_b): the first arrival in the block
//   G_b  = -log_det(E_b)                ~ Gumbel(log n_b): the block's MAX noise
//   p_b  = (wb * n_b) >> 32             uniform position of that maximum
// Every other element v of the block gets a Gumbel truncated below G_b:
//   A_v  = -log_det(u(w_v)),  w_v = word (v & 3) of Philox(v >> 2, pos, seq_lo, seq_hi)
//   g_v  = min(G_b, -log_det(RN(E_b + A_v)))      (= -log(e^{-G_b} + Exp(1)))
// and g_{p_b} = G_b.  (In exact arithmetic g_v < G_b already; the min makes the
// block bound g_v <= G_b hold under rounding too.)  All counters depend on
// (seed, seq_id, pos, v) only, so rows at the same position share noise.
constexpr int64_t BLK = 64;

void row_noise(int64_t V, uint64_t seed, uint64_t seq_id, int32_t pos, float* g) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const uint32_t slo = (uint32_t)seq_id, shi = (uint32_t)(seq_id >> 32);
  const int64_t nblk = (V + BLK - 1) / BLK;
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t v0 = b * BLK;
    const uint32_t n = (uint32_t)std::min<int64_t>(BLK, V - v0);
    uint32_t bctr[4] = {0x80000000u | (uint32_t)(b >> 1), (uint32_t)pos, slo, shi};
    uint32_t bw[4];
    philox4x32_10(bctr, key, bw);
    const uint32_t wa = (b & 1) ? bw[2] : bw[0];
    const uint32_t wb = (b & 1) ? bw[3] : bw[1];
    const float a = -log_det(uniform_from_word(wa));
    const float E = a / (float)n;
    const float G = -log_det(E);
    const uint32_t p = (uint32_t)(((uint64_t)wb * n) >> 32);
    for (uint32_t j = 0; j < n; ++j) {
      const int64_t v = v0 + j;
      if (j == p) {
        g[v] = G;
        continue;
      }
      uint32_t ctr[4] = {(uint32_t)(v >> 2), (uint32_t)pos, slo, shi};
      uint32_t out[4];
      philox4x32_10(ctr, key, out);
      const float A = -log_det(uniform_from_word(out[v & 3]));
      const float Tv = E + A;
      const float gv = -log_det(Tv);
      g[v] = gv > G ? G : gv;
    }
  }
}

// One logits row -> the sampled token (reading O11, BJ:north_star part 4):
//   tau = argmax_v  RN32( RN32(x_v / T) + g_v ),   g_v from row_noise above,
//   first (smallest) index on ties; NaN logits are not candidates (flagged);
//   if there is no candidate at all the result is 0.
// ties (nullable) receives the number of indices whose z equals the maximum
// (>= 2: a float tie, decided by the smallest-index rule; north_star's tie count).
int32_t sample_row(const void* row, int dtype, int64_t V, uint64_t seed, uint64_t seq_id,
                   int32_t pos, float temperature, int* nan_seen, int32_t* ties = nullptr) {
  std::vector<float> noise((size_t)V);
  row_noise(V, seed, seq_id, pos, noise.data());
  int32_t best = 0;
  float best_z = 0.0f;
  bool have = false;
  int32_t n_best = 0;
  for (int64_t v = 0; v < V; ++v) {
    const float g = noise[(size_t)v];
    float x = load_logit(row, dtype, v);
    if (std::isnan(x)) {
      *nan_seen = 1;
      continue;
    }
    if (temperature != 1.0f) x = x / temperature;
    float z = x + g;
    if (!have || z > best_z) {
      best_z = z;
      best = (int32_t)v;
      have = true;
      n_best = 1;
    } else if (z == best_z) {
      ++n_best;
    }
  }
  if (ties) *ties = n_best;
  return best;
}

// ---------------------------------------------------------------------------
// Insert ("index all substrings", "inserted online"; reading O1/O2):
// for every window start i in [max(floor, from-D+1), to), walk the root along
// tokens[i .. min(i+D, to)-1], creating missing nodes; the node reached after
// consuming tokens[i..j] gets +1 iff j >= from (a window ending at a new
// position).  After all inserts, count(u) = number of occurrences of u's
// string that end at an inserted position.
// ---------------------------------------------------------------------------
void insert_span(Cache* c, int32_t p, const int32_t* toks, int32_t from, int32_t to,
                 int32_t floor_) {
  const int32_t D = c->cfg.max_depth;
  if (p < 0 || p >= c->cfg.max_prompts) {
    c->error_bits |= 4u;
    return;
  }
  int32_t lo = std::max(floor_, from - D + 1);
  if (lo < 0) lo = 0;
  for (int32_t i = lo; i < to; ++i) {
    Node* u = c->roots[p].get();
    int32_t end = std::min(i + D, to);
    for (int32_t j = i; j < end; ++j) {
      int32_t tok = toks[j];
      if (tok < 0 || tok >= c->cfg.vocab_size) {
        c->error_bits |= 1u;
        break;
      }
      u = child_or_create(c, u, tok);
      if (j >= from) u->count += 1;
    }
  }
}

// ---------------------------------------------------------------------------
// Longest-suffix match (reading O3): the largest q in [1, min(L, t)]
// such that walking the root along y[t-q .. t-1] succeeds AND the reached node
// has at least one child; q = 0 (fallback) if none.
// ---------------------------------------------------------------------------
int32_t match(Cache* c, int32_t p, const int32_t* y, int32_t t, Node** u_out) {
  int32_t best_q = 0;
  Node* best_u = nullptr;
  int32_t qmax = std::min(c->cfg.max_match_len, t);
  for (int32_t q = 1; q <= qmax; ++q) {
    Node* u = c->roots[p].get();
    for (int32_t j = t - q; j < t && u != nullptr; ++j) u = find_child(u, y[j]);
    if (u != nullptr && !u->kids.empty()) {
      best_q = q;
      best_u = u;
    }
  }
  *u_out = best_u;
  return best_q;
}

// ---------------------------------------------------------------------------
// Best-first draft (readings O4-O9).
// C(v) = count(v) / sum_{w in children(parent(v))} count(w)    (fp64 RN)
// score(v) = score(parent) * C(v), score(u_q) = 1               (fp64 RN)
// Pop the frontier maximum under the total order O8 (score desc, depth asc,
// token asc, parent's draft index asc) until B(q) nodes are drafted, the
// frontier is empty, or the best score < min_path_score.
// ---------------------------------------------------------------------------
struct Cand {
  double score;
  int32_t depth;   // relative to u_q (children of u_q have depth 1)
  int32_t tok;
  int32_t parent;  // draft index of the parent, -1 for u_q
  Node* node;
};

bool better(const Cand& a, const Cand& b) {
  if (a.score != b.score) return a.score > b.score;
  if (a.depth != b.depth) return a.depth < b.depth;
  if (a.tok != b.tok) return a.tok < b.tok;
  return a.parent < b.parent;
}

struct WorseFirst {  // priority_queue puts the element that is NOT worse on top
  bool operator()(const Cand& a, const Cand& b) const { return better(b, a); }
};

void push_children(std::priority_queue<Cand, std::vector<Cand>, WorseFirst>& pq, Node* u,
                   double score_u, int32_t depth_u, int32_t parent_idx) {
  uint64_t sum = 0;
  for (auto& kv : u->kids) sum += kv.second->count;
  for (auto& kv : u->kids) {
    double C = (sum == 0) ? 0.0 : (double)kv.second->count / (double)sum;
    double score = score_u * C;
    pq.push(Cand{score, depth_u + 1, kv.first, parent_idx, kv.second.get()});
  }
}

int32_t budget(const Config& cfg, int32_t q) {
  int64_t b = (int64_t)cfg.budget_base + ((int64_t)q * cfg.budget_slope_num) / cfg.budget_slope_den;
  return (int32_t)std::min<int64_t>(cfg.budget_max, b);
}

}  // namespace

// =============================================================================
// C ABI (host pointers only).  Mirrors the GPU library's calls one for one so
// that a test can feed both the same arrays.
// =============================================================================
extern "C" {

int orc_abi_version() { return 1; }

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox4x32_10(ctr, key, out);
}

float orc_log_det(float x) { return log_det(x); }

void orc_log_det_array(const float* x, float* out, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = log_det(x[i]);
}

float orc_gumbel_from_word(uint32_t w) { return gumbel_from_word(w); }

// g(r) for every r in [0, 2^23): the whole noise domain (pin P9).
void orc_noise_table(float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (1 << 23); ++r) out[r] = gumbel_from_word((uint32_t)r << 9);
}

// g_v for every v of one row key (the noise of the sampler; test support).
void orc_row_noise(int64_t V, uint64_t seed, uint64_t seq_id, int32_t pos, float* g) {
  row_noise(V, seed, seq_id, pos, g);
}

int32_t orc_sample_row(const void* row, int dtype, int64_t V, uint64_t seed, uint64_t seq_id,
                       int32_t pos, float temperature, int* nan_seen) {
  return sample_row(row, dtype, V, seed, seq_id, pos, temperature, nan_seen);
}

// The noise of n row keys (seq_id[k], pos[k]) into out[k*V ...], one key per
// thread (test support: the element-level GPU comparison).
void orc_row_noise_many(int64_t V, uint64_t seed, int32_t n, const uint64_t* seq_id,
                        const int32_t* pos, float* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t k = 0; k < n; ++k) row_noise(V, seed, seq_id[k], pos[k], out + (int64_t)k * V);
}

// sample_row over n independent rows (rows[k*V ...], key (seq_id[k], pos[k])),
// one row per thread: tok[k], ties[k] (indices sharing the maximum z), nan[k].
void orc_sample_rows(const void* rows, int dtype, int64_t V, int32_t n, uint64_t seed,
                     const uint64_t* seq_id, const int32_t* pos, float temperature, int32_t* tok,
                     int32_t* ties, int32_t* nan_seen) {
  const int64_t esz = dtype == 0 ? 2 : 4;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t k = 0; k < n; ++k) {
    int nan = 0;
    tok[k] = sample_row((const char*)rows + (int64_t)k * V * esz, dtype, V, seed, seq_id[k], pos[k],
                        temperature, &nan, &ties[k]);
    nan_seen[k] = nan;
  }
}

void* orc_cache_create(int32_t vocab_size, int32_t max_prompts, int32_t max_depth,
                       int32_t max_match_len, int32_t budget_max, int32_t budget_base,
                       int32_t slope_num, int32_t slope_den, double min_path_score) {
  if (vocab_size < 2 || max_prompts < 1 || max_depth < 1 || max_match_len < 1 ||
      max_match_len > max_depth || budget_max < 1 || budget_max > 64 || budget_base < 0 ||
      budget_base > budget_max || slope_num < 0 || slope_den < 1)
    return nullptr;
  Cache* c = new Cache();
  c->cfg = Config{vocab_size, max_prompts, max_depth, max_match_len, budget_max,
                  budget_base, slope_num, slope_den, min_path_score};
  c->roots.resize(max_prompts);
  for (auto& r : c->roots) r = std::make_unique<Node>();
  return c;
}

void orc_cache_destroy(void* h) { delete (Cache*)h; }

uint32_t orc_error_bits(void* h) { return ((Cache*)h)->error_bits; }
uint64_t orc_node_count(void* h) { return ((Cache*)h)->nodes; }

// Batched insert: span s = (prompt_id[s], seq_tok[s*stride ...], [from[s], to[s]), floor[s]).
// Spans are applied in index order (counts commute, so order is unobservable).
void orc_insert(void* h, int32_t n, const int32_t* prompt_id, const int32_t* seq_tok,
                int64_t stride, const int32_t* from, const int32_t* to, const int32_t* floor_) {
  Cache* c = (Cache*)h;
  for (int32_t s = 0; s < n; ++s)
    insert_span(c, prompt_id[s], seq_tok + (int64_t)s * stride, from[s], to[s],
                floor_ ? floor_[s] : 0);
}

// Batched draft (match + best-first + layout).  Output arrays per sequence s
// have Bmax entries (draft_*) ; unused entries are tok=-1, parent=-1, depth=0,
// pos=-1, mask=0.  row_offsets[n+1] = exclusive scan of (draft_len + 1)
// (logits row order per sequence: [root, node 0, ..., node n_s-1], O9).
void orc_draft(void* h, int32_t n, const int32_t* prompt_id, const int32_t* seq_tok,
               int64_t stride, const int32_t* seq_len, const int32_t* pos_base,
               int32_t* match_len, int32_t* draft_len, int32_t* draft_tok, int32_t* draft_parent,
               int32_t* draft_depth, int32_t* draft_pos, uint64_t* draft_mask,
               int64_t* row_offsets) {
  Cache* c = (Cache*)h;
  const int32_t Bmax = c->cfg.budget_max;
  row_offsets[0] = 0;
  for (int32_t s = 0; s < n; ++s) {
    int32_t* dtok = draft_tok + (int64_t)s * Bmax;
    int32_t* dpar = draft_parent + (int64_t)s * Bmax;
    int32_t* ddep = draft_depth + (int64_t)s * Bmax;
    int32_t* dpos = draft_pos + (int64_t)s * Bmax;
    uint64_t* dmask = draft_mask + (int64_t)s * Bmax;
    for (int32_t i = 0; i < Bmax; ++i) {
      dtok[i] = -1; dpar[i] = -1; ddep[i] = 0; dpos[i] = -1; dmask[i] = 0;
    }
    int32_t p = prompt_id[s];
    int32_t q = 0;
    Node* u = nullptr;
    if (p >= 0 && p < c->cfg.max_prompts)
      q = match(c, p, seq_tok + (int64_t)s * stride, seq_len[s], &u);
    else
      c->error_bits |= 4u;
    int32_t ndraft = 0;
    if (q > 0) {
      int32_t B = budget(c->cfg, q);
      std::priority_queue<Cand, std::vector<Cand>, WorseFirst> pq;
      push_children(pq, u, 1.0, 0, -1);
      while (ndraft < B && !pq.empty()) {
        Cand top = pq.top();
        if (top.score < c->cfg.min_path_score) break;
        pq.pop();
        int32_t i = ndraft++;
        dtok[i] = top.tok;
        dpar[i] = top.parent;
        ddep[i] = top.depth;
        dpos[i] = pos_base[s] + top.depth;
        dmask[i] = (top.parent >= 0 ? dmask[top.parent] : 0ull) | (1ull << i);
        push_children(pq, top.node, top.score, top.depth, i);
      }
    }
    match_len[s] = q;
    draft_len[s] = ndraft;
    row_offsets[s + 1] = row_offsets[s] + ndraft + 1;
  }
}

// Batched verify: sample every row (root + each draft node), then walk the
// draft accepting up to the first mismatch and commit tau along the path
// (accepted tokens + 1 bonus), truncated after the first EOS (inclusive) or at
// max_new (readings O10, O13).  Appends to the sequence table.
// Row r = row_offsets[s] is the root of sequence s (position t = seq_len[s]);
// row row_offsets[s]+1+i is draft node i (position t + draft_depth[i]).
// ties (nullable): per row, the number of indices sharing the maximum z.
// Returns 1 if a NaN logit was seen.
int orc_verify(void* h, int32_t n, const void* logits, int dtype, const int64_t* row_offsets,
               const int32_t* draft_len, const int32_t* draft_tok, const int32_t* draft_parent,
               const int32_t* draft_depth, const uint64_t* seq_id, uint64_t seed,
               float temperature, int32_t eos_id, const int32_t* max_new, int32_t* seq_tok,
               int64_t stride, int32_t* seq_len, int32_t* sampled, int32_t* accept_len,
               int32_t* n_commit, int32_t* commit_tok, int32_t* accepted_nodes, uint8_t* finished,
               int32_t* ties) {
  Cache* c = (Cache*)h;
  const int32_t Bmax = c->cfg.budget_max;
  const int64_t V = c->cfg.vocab_size;
  int nan_any = 0;
  // 1) sample every row
#pragma omp parallel for schedule(dynamic, 1) reduction(| : nan_any)
  for (int32_t s = 0; s < n; ++s) {
    int32_t t = seq_len[s];
    for (int32_t i = -1; i < draft_len[s]; ++i) {
      int64_t r = row_offsets[s] + 1 + i;
      int32_t pos = t + (i < 0 ? 0 : draft_depth[(int64_t)s * Bmax + i]);
      const char* row = (const char*)logits + r * V * (dtype == 0 ? 2 : 4);
      int nan_seen = 0;
      int32_t nt = 0;
      sampled[r] = sample_row(row, dtype, V, seed, seq_id[s], pos, temperature, &nan_seen, &nt);
      if (ties) ties[r] = nt;
      nan_any |= nan_seen;
    }
  }
  // 2) walk + commit
  for (int32_t s = 0; s < n; ++s) {
    const int32_t* dtok = draft_tok + (int64_t)s * Bmax;
    const int32_t* dpar = draft_parent + (int64_t)s * Bmax;
    int32_t* acc = accepted_nodes + (int64_t)s * Bmax;
    int32_t* com = commit_tok + (int64_t)s * (Bmax + 1);
    for (int32_t i = 0; i < Bmax; ++i) acc[i] = -1;
    for (int32_t i = 0; i < Bmax + 1; ++i) com[i] = -1;
    int32_t cur = -1;  // -1 = the draft root (last committed token)
    int32_t a = 0;
    std::vector<int32_t> path_tokens;
    while (true) {
      int32_t tau = sampled[row_offsets[s] + 1 + cur];
      path_tokens.push_back(tau);
      int32_t next = -1;
      for (int32_t i = 0; i < draft_len[s]; ++i)
        if (dpar[i] == cur && dtok[i] == tau) { next = i; break; }
      if (next < 0) break;
      acc[a++] = next;
      cur = next;
    }
    int32_t t = seq_len[s];
    int32_t nc = (int32_t)path_tokens.size();  // a + 1
    int32_t cap = max_new[s] - t;
    if (cap < 0) cap = 0;
    if (nc > cap) nc = cap;
    bool hit_eos = false;
    if (eos_id >= 0)
      for (int32_t k = 0; k < nc; ++k)
        if (path_tokens[k] == eos_id) { nc = k + 1; hit_eos = true; break; }
    for (int32_t k = 0; k < nc; ++k) {
      com[k] = path_tokens[k];
      seq_tok[(int64_t)s * stride + t + k] = path_tokens[k];
    }
    accept_len[s] = a;
    n_commit[s] = nc;
    seq_len[s] = t + nc;
    finished[s] = (hit_eos || seq_len[s] >= max_new[s]) ? 1 : 0;
  }
  return nan_any;
}

// Canonical dump of T_p (SPEC S:L148-149 format): preorder records
// (token, count, n_children), children in ascending token order.  The root
// record is (-1, sum of depth-1 counts, n_children).  Returns the number of
// records (writes at most cap of them).
int64_t orc_dump(void* h, int32_t p, int32_t* tok, uint64_t* count, int32_t* nchild, int64_t cap) {
  Cache* c = (Cache*)h;
  if (p < 0 || p >= c->cfg.max_prompts) return -1;
  int64_t k = 0;
  std::vector<Node*> stack;
  Node* root = c->roots[p].get();
  uint64_t rootsum = 0;
  for (auto& kv : root->kids) rootsum += kv.second->count;
  stack.push_back(root);
  while (!stack.empty()) {
    Node* u = stack.back();
    stack.pop_back();
    if (k < cap) {
      tok[k] = (u == root) ? -1 : u->tok;
      count[k] = (u == root) ? rootsum : u->count;
      nchild[k] = (int32_t)u->kids.size();
    }
    ++k;
    for (auto it = u->kids.rbegin(); it != u->kids.rend(); ++it) stack.push_back(it->second.get());
  }
  return k;
}

// ---------------------------------------------------------------------------
// Capacity management (reading O17 in DESIGN.md).  The paper
// bounds nothing ("can be stored in CPU memory"); SPEC's evict
// removes whole subtrees in ascending count order.  Reading:
// prune(p, theta) removes every non-root node whose count is below theta.
// Because count(u) >= the count of each child (O1), that set is closed under
// descendants, so exactly whole subtrees go, lowest counts first.
// ---------------------------------------------------------------------------
static uint64_t prune_node(Node* u, uint64_t theta) {
  uint64_t removed = 0;
  for (auto it = u->kids.begin(); it != u->kids.end();) {
    if (it->second->count < theta) {
      std::vector<Node*> stack = {it->second.get()};  // count the subtree
      while (!stack.empty()) {
        Node* v = stack.back();
        stack.pop_back();
        ++removed;
        for (auto& kv : v->kids) stack.push_back(kv.second.get());
      }
      it = u->kids.erase(it);
    } else {
      removed += prune_node(it->second.get(), theta);
      ++it;
    }
  }
  return removed;
}

// Remove every non-root node of T_p (every p if p < 0) with count < theta.
// Returns the number of nodes removed.
int64_t orc_prune(void* h, int32_t p, uint64_t theta) {
  Cache* c = (Cache*)h;
  if (p >= c->cfg.max_prompts) return -1;
  uint64_t removed = 0;
  for (int32_t q = 0; q < c->cfg.max_prompts; ++q)
    if (p < 0 || q == p) removed += prune_node(c->roots[q].get(), theta);
  c->nodes -= removed;
  return (int64_t)removed;
}

// Merge a canonical dump (orc_dump's records, preorder) into T_p: every
// record's path is created if missing and its count added.  Loading a dump
// into an empty tree reproduces it exactly (persistence across training
// steps).  Returns 0, or -1 for a malformed record list.
int32_t orc_load(void* h, int32_t p, const int32_t* tok, const uint64_t* count,
                 const int32_t* nchild, int64_t n) {
  Cache* c = (Cache*)h;
  if (p < 0 || p >= c->cfg.max_prompts || n < 1 || tok[0] != -1) return -1;
  // (node, children still to read) along the current preorder path
  std::vector<std::pair<Node*, int32_t>> path = {{c->roots[p].get(), nchild[0]}};
  for (int64_t k = 1; k < n; ++k) {
    while (!path.empty() && path.back().second == 0) path.pop_back();
    if (path.empty()) return -1;
    path.back().second -= 1;
    Node* v = child_or_create(c, path.back().first, tok[k]);
    v->count += count[k];
    path.push_back({v, nchild[k]});
  }
  return 0;
}

// Count of a string (root walk), 0 if absent.  Test helper.
uint64_t orc_count_of(void* h, int32_t p, const int32_t* toks, int32_t len) {
  Cache* c = (Cache*)h;
  Node* u = c->roots[p].get();
  for (int32_t j = 0; j < len && u; ++j) u = find_child(u, toks[j]);
  return u ? u->count : 0;
}

}  // extern "C"
