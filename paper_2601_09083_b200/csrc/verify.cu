// verify.cu — srt_verify: Gumbel-max sample at every draft row, then the
// first-mismatch walk and commit (readings O10, O11, O13).
//
// The scan is the roofline kernel: it reads every logits row once and is
// HBM-bound by design (no tensor cores: nothing here is a contraction).  The
// plain definition costs ~60 instructions per element (Philox4x32-10 + two
// IEEE-division logs), far above the ~13 per element the HBM roofline allows,
// so the product scan is EXACTLY pruned:
//   1. row max X and its first index i*; M_lb = z(i*) computed exactly;
//   2. z_v = RN(RN(x_v/T) + g_v) <= RN(RN(x_v/T) + gmax): skip v if that is < M,
//      where M >= M_lb is an achieved z (so a skipped v can neither win nor tie);
//   3. for survivors, Philox once per quad, then the per-bucket bound
//      RN(RN(x/T) + G[r >> 13]) < M skips the two logs; else z exactly.
// The unpruned kernel (srt_sample_rows_reference) evaluates every element and
// is kept to show the pruning changes no bit.
#include <cuda_bf16.h>

#include "noise.cuh"
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int REF_THREADS = 256;

struct RowMeta {
  int64_t row;
  int32_t seq;
  int32_t pos;
  uint32_t sid_lo, sid_hi;
};

__device__ __forceinline__ RowMeta row_meta(const VerifyArgs& a, int32_t Bmax, int64_t r) {
  int32_t lo = 0, hi = a.n - 1;  // last s with row_offsets[s] <= r
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (a.row_offsets[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const int32_t s = lo;
  const int64_t node = r - a.row_offsets[s] - 1;  // -1 = root
  const int32_t pos = a.seq_len[s] + (node < 0 ? 0 : a.draft_depth[(int64_t)s * Bmax + node]);
  const uint64_t sid = a.seq_id[s];
  return RowMeta{r, s, pos, (uint32_t)sid, (uint32_t)(sid >> 32)};
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float load_elem(const void* row, int dtype, int64_t v) {
  if (dtype == SRT_BF16) {
    const uint16_t h = ((const uint16_t*)row)[v];
    return __uint_as_float((uint32_t)h << 16);
  }
  return ((const float*)row)[v];
}

__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

// Block-wide reduction of (z, v) candidates under cand_better.
template <int THREADS>
__device__ __forceinline__ void block_argmax(float& bz, int32_t& bv, float* sz, int32_t* sv) {
  for (int o = 16; o; o >>= 1) {
    const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
    const int32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
    if (cand_better(oz, ov, bz, bv)) { bz = oz; bv = ov; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sz[w] = bz; sv[w] = bv; }
  __syncthreads();
  if (w == 0) {
    bz = lane < THREADS / 32 ? sz[lane] : -INFINITY;
    bv = lane < THREADS / 32 ? sv[lane] : INT_MAX;
    for (int o = 16; o; o >>= 1) {
      const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
      const int32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
      if (cand_better(oz, ov, bz, bv)) { bz = oz; bv = ov; }
    }
  }
}

// ---------------------------------------------------------------------------
// Reference scan: every element evaluated (the plain definition on the GPU).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(REF_THREADS) k_scan_reference(DevCache c, VerifyArgs a) {
  __shared__ float sz[REF_THREADS / 32];
  __shared__ int32_t sv[REF_THREADS / 32];
  __shared__ RowMeta meta;
  const int64_t total = a.row_offsets[a.n];
  const int64_t V = c.V;
  const size_t esz = a.dtype == SRT_BF16 ? 2 : 4;
  const bool unit_t = a.temperature == 1.0f;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  for (int64_t r = blockIdx.x; r < total; r += gridDim.x) {
    if (threadIdx.x == 0) meta = row_meta(a, c.Bmax, r);
    __syncthreads();
    const RowMeta m = meta;
    const char* row = (const char*)a.logits + r * V * esz;
    float bz = -INFINITY;
    int32_t bv = INT_MAX;
    bool nan_seen = false;
    for (int64_t qd = threadIdx.x; qd * 4 < V; qd += REF_THREADS) {
      const Philox4 w = philox4x32_10((uint32_t)qd, (uint32_t)m.pos, m.sid_lo, m.sid_hi, k0, k1);
      const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t v = qd * 4 + k;
        if (v >= V) break;
        const float x = load_elem(row, a.dtype, v);
        if (x != x) { nan_seen = true; continue; }
        const float z = perturbed(x, gumbel_of_r(words[k] >> 9), a.temperature, unit_t);
        if (cand_better(z, (int32_t)v, bz, bv)) { bz = z; bv = (int32_t)v; }
      }
    }
    if (nan_seen) set_error(c, SRT_DEV_NONFINITE_LOGIT);
    block_argmax<REF_THREADS>(bz, bv, sz, sv);
    if (threadIdx.x == 0) a.sampled[r] = bv == INT_MAX ? 0 : bv;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Pruned scan, one CTA per row, 16-byte vector loads (8 bf16 or 4 f32).
// Pass 1 streams the row from HBM (max + NaN detection); pass 2 re-reads it
// (L2-resident: <= 1 row per SM in flight) and evaluates only survivors.
// Requires V*esz % 16 == 0 and a 16-byte aligned base; otherwise the
// reference kernel is used.
// ---------------------------------------------------------------------------
template <int DT>
struct Vec;
template <>
struct Vec<SRT_BF16> {
  static constexpr int E = 8;
  __device__ __forceinline__ static void unpack(const uint4& q, float x[8]) {
    x[0] = bf16_lo(q.x); x[1] = bf16_hi(q.x); x[2] = bf16_lo(q.y); x[3] = bf16_hi(q.y);
    x[4] = bf16_lo(q.z); x[5] = bf16_hi(q.z); x[6] = bf16_lo(q.w); x[7] = bf16_hi(q.w);
  }
  // NaN-propagating max of the 8 values (packed bf16x2)
  __device__ __forceinline__ static float vmax_nan(const uint4& q) {
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&q.x);
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&q.y);
    __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&q.z);
    __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&q.w);
    __nv_bfloat162 m = __hmax2_nan(__hmax2_nan(a, b), __hmax2_nan(c, d));
    return max_nan(__low2float(m), __high2float(m));
  }
  __device__ __forceinline__ static float vmax(const uint4& q) {
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&q.x);
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&q.y);
    __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&q.z);
    __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&q.w);
    __nv_bfloat162 m = __hmax2(__hmax2(a, b), __hmax2(c, d));
    return fmaxf(__low2float(m), __high2float(m));
  }
};
template <>
struct Vec<SRT_F32> {
  static constexpr int E = 4;
  __device__ __forceinline__ static void unpack(const uint4& q, float x[4]) {
    x[0] = __uint_as_float(q.x); x[1] = __uint_as_float(q.y);
    x[2] = __uint_as_float(q.z); x[3] = __uint_as_float(q.w);
  }
  __device__ __forceinline__ static float vmax_nan(const uint4& q) {
    return max_nan(max_nan(__uint_as_float(q.x), __uint_as_float(q.y)),
                   max_nan(__uint_as_float(q.z), __uint_as_float(q.w)));
  }
  __device__ __forceinline__ static float vmax(const uint4& q) {
    return fmaxf(fmaxf(__uint_as_float(q.x), __uint_as_float(q.y)),
                 fmaxf(__uint_as_float(q.z), __uint_as_float(q.w)));
  }
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int DT>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_pruned(DevCache c, VerifyArgs a) {
  using VT = Vec<DT>;
  constexpr int E = VT::E;
  __shared__ float sgb[NOISE_BUCKETS];
  __shared__ float sz[SCAN_THREADS / 32];
  __shared__ int32_t sv[SCAN_THREADS / 32];
  __shared__ RowMeta meta;
  __shared__ float s_x;        // row max
  __shared__ int32_t s_istar;  // its first index
  __shared__ float s_mlb;      // z(i*)
  for (int i = threadIdx.x; i < NOISE_BUCKETS; i += SCAN_THREADS) sgb[i] = c.gbound[i];
  const float gmax = c.gbound[NOISE_BUCKETS];
  const int64_t total = a.row_offsets[a.n];
  const int64_t V = c.V;
  const int64_t nvec = V / E;
  const bool unit_t = a.temperature == 1.0f;
  const float T = a.temperature;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t r = blockIdx.x; r < total; r += gridDim.x) {
    if (threadIdx.x == 0) meta = row_meta(a, c.Bmax, r);
    const uint4* row = (const uint4*)((const char*)a.logits + r * V * (DT == SRT_BF16 ? 2 : 4));
    // ---- pass 1: NaN-propagating max, first vector achieving it per thread
    float tmax = -INFINITY;
    int64_t tvec = -1;
    bool has_nan = false;
    for (int64_t j = threadIdx.x; j < nvec; j += SCAN_THREADS) {
      const float m = VT::vmax_nan(ldg_stream(row + j));
      if (m != m) { has_nan = true; break; }
      if (m > tmax || tvec < 0) { tmax = m; tvec = j; }
    }
    has_nan = __syncthreads_or(has_nan);
    if (has_nan) {  // rare: flag, then recompute the max ignoring NaNs
      if (threadIdx.x == 0) set_error(c, SRT_DEV_NONFINITE_LOGIT);
      tmax = -INFINITY;
      tvec = -1;
      for (int64_t j = threadIdx.x; j < nvec; j += SCAN_THREADS) {
        const float m = VT::vmax(ldg_stream(row + j));  // NaN only if all 8 are NaN
        if (m == m && (m > tmax || tvec < 0)) { tmax = m; tvec = j; }
      }
    }
    // block max
    float bm = tmax;
    for (int o = 16; o; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
    if (lane == 0) sz[wid] = bm;
    __syncthreads();
    if (threadIdx.x < 32) {
      float x = threadIdx.x < SCAN_THREADS / 32 ? sz[threadIdx.x] : -INFINITY;
      for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (threadIdx.x == 0) { s_x = x; s_istar = INT_MAX; }
    }
    __syncthreads();
    const float X = s_x;
    if (X == X && tvec >= 0 && tmax == X) {  // find the first element equal to X
      float xs[E];
      VT::unpack(ldg_stream(row + tvec), xs);
      int32_t first = INT_MAX;
#pragma unroll
      for (int k = E - 1; k >= 0; --k)
        if (xs[k] == X) first = (int32_t)(tvec * E + k);
      atomicMin(&s_istar, first);
    }
    __syncthreads();
    const RowMeta m = meta;
    if (threadIdx.x == 0) {
      float mlb = NAN;
      const int32_t is = s_istar;
      if (is != INT_MAX) {
        const Philox4 w =
            philox4x32_10((uint32_t)(is >> 2), (uint32_t)m.pos, m.sid_lo, m.sid_hi, k0, k1);
        const uint32_t wk = (is & 3) == 0 ? w.x : (is & 3) == 1 ? w.y : (is & 3) == 2 ? w.z : w.w;
        mlb = perturbed(X, gumbel_of_r(wk >> 9), T, unit_t);
      }
      s_mlb = mlb;
    }
    __syncthreads();
    // ---- pass 2: survivors only
    float bz = -INFINITY;
    int32_t bv = INT_MAX;
    const float mlb = s_mlb;
    if (mlb == mlb) {  // at least one non-NaN element
      float M = mlb;
      for (int64_t j = threadIdx.x; j < nvec; j += SCAN_THREADS) {
        const uint4 q = ldg_stream(row + j);
        const float vm = VT::vmax(q);
        const float vms = unit_t ? vm : __fdiv_rn(vm, T);
        if (!(__fadd_rn(vms, gmax) >= M)) continue;  // whole vector pruned (NaN-safe)
        float xs[E];
        VT::unpack(q, xs);
#pragma unroll
        for (int qq = 0; qq < E / 4; ++qq) {
          float xq[4];
          unsigned sv_mask = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            xq[k] = unit_t ? xs[qq * 4 + k] : __fdiv_rn(xs[qq * 4 + k], T);
            if (__fadd_rn(xq[k], gmax) >= M) sv_mask |= 1u << k;
          }
          if (!sv_mask) continue;
          const int64_t v0 = j * E + qq * 4;
          const Philox4 w =
              philox4x32_10((uint32_t)(v0 >> 2), (uint32_t)m.pos, m.sid_lo, m.sid_hi, k0, k1);
          const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (!(sv_mask & (1u << k))) continue;
            const uint32_t rr = words[k] >> 9;
            if (__fadd_rn(xq[k], sgb[rr >> NOISE_BUCKET_SHIFT]) < M) continue;
            const float z = __fadd_rn(xq[k], gumbel_of_r(rr));
            if (cand_better(z, (int32_t)(v0 + k), bz, bv)) {
              bz = z;
              bv = (int32_t)(v0 + k);
              M = fmaxf(M, z);
            }
          }
        }
      }
    }
    block_argmax<SCAN_THREADS>(bz, bv, sz, sv);
    if (threadIdx.x == 0) a.sampled[r] = bv == INT_MAX ? 0 : bv;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Accept + commit: one warp per sequence.
// ---------------------------------------------------------------------------
constexpr int ACC_WARPS = 4;

__global__ void __launch_bounds__(ACC_WARPS * 32) k_accept(DevCache c, VerifyArgs a) {
  __shared__ int32_t ctok[ACC_WARPS][65];
  __shared__ int32_t acc[ACC_WARPS][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * ACC_WARPS + w;
  if (s >= a.n) return;
  const int32_t B = c.Bmax;
  const int32_t ns = a.draft_len[s];
  const int64_t r0 = a.row_offsets[s];
  const int32_t t = a.seq_len[s];
  const int64_t db = (int64_t)s * B;
  const bool vA = lane < ns, vB = lane + 32 < ns;
  const int32_t tokA = vA ? a.draft_tok[db + lane] : -1;
  const int32_t parA = vA ? a.draft_parent[db + lane] : -2;
  const int32_t smpA = vA ? a.sampled[r0 + 1 + lane] : 0;
  const int32_t tokB = vB ? a.draft_tok[db + lane + 32] : -1;
  const int32_t parB = vB ? a.draft_parent[db + lane + 32] : -2;
  const int32_t smpB = vB ? a.sampled[r0 + 33 + lane] : 0;
  const int32_t root = a.sampled[r0];
  int32_t cur = -1, na = 0;
  while (true) {
    const int32_t sa = __shfl_sync(0xffffffffu, smpA, cur & 31);
    const int32_t sb = __shfl_sync(0xffffffffu, smpB, cur & 31);
    const int32_t tau = cur < 0 ? root : (cur < 32 ? sa : sb);
    if (lane == 0) ctok[w][na] = tau;
    const unsigned m0 = __ballot_sync(0xffffffffu, vA && parA == cur && tokA == tau);
    const unsigned m1 = __ballot_sync(0xffffffffu, vB && parB == cur && tokB == tau);
    const int32_t next = m0 ? __ffs(m0) - 1 : (m1 ? 31 + __ffs(m1) : -1);
    if (next < 0 || na >= B) break;
    if (lane == 0) acc[w][na] = next;
    ++na;
    cur = next;
  }
  __syncwarp();
  int32_t nc = na + 1;
  const int32_t cap = max(0, a.max_new[s] - t);
  nc = min(nc, cap);
  bool hit = false;
  if (a.eos_id >= 0) {
    int32_t first = INT_MAX;
    for (int32_t k = lane; k < nc; k += 32)
      if (ctok[w][k] == a.eos_id) first = min(first, k);
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (first != INT_MAX) { nc = first + 1; hit = true; }
  }
  for (int32_t k = lane; k < B + 1; k += 32) {
    const int32_t v = k < nc ? ctok[w][k] : -1;
    a.commit_tok[(int64_t)s * (B + 1) + k] = v;
    if (k < nc) a.seq_tok[(int64_t)s * a.stride + t + k] = v;
  }
  for (int32_t k = lane; k < B; k += 32) a.accepted_nodes[db + k] = k < na ? acc[w][k] : -1;
  if (lane == 0) {
    a.accept_len[s] = na;
    a.n_commit[s] = nc;
    a.seq_len[s] = t + nc;
    a.finished[s] = (hit || t + nc >= a.max_new[s]) ? 1 : 0;
  }
}

}  // namespace

cudaError_t launch_scan(const DevCache& c, const VerifyArgs& a, bool reference,
                        cudaStream_t stream) {
  const size_t esz = a.dtype == SRT_BF16 ? 2 : 4;
  const bool vec_ok = ((size_t)c.V * esz) % 16 == 0 && ((uintptr_t)a.logits % 16) == 0;
  if (reference || !vec_ok) {
    k_scan_reference<<<num_sms() * 8, REF_THREADS, 0, stream>>>(c, a);
  } else if (a.dtype == SRT_BF16) {
    k_scan_pruned<SRT_BF16><<<num_sms() * 2, SCAN_THREADS, 0, stream>>>(c, a);
  } else {
    k_scan_pruned<SRT_F32><<<num_sms() * 2, SCAN_THREADS, 0, stream>>>(c, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_accept(const DevCache& c, const VerifyArgs& a, cudaStream_t stream) {
  k_accept<<<(a.n + ACC_WARPS - 1) / ACC_WARPS, ACC_WARPS * 32, 0, stream>>>(c, a);
  return cudaGetLastError();
}

}  // namespace srt
