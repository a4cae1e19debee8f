// verify.cu — srt_verify: Gumbel-max sample at every draft row, then the
// first-mismatch walk and commit (readings O10, O11, O13).
//
// The scan is the roofline kernel (scan.cu: cluster/TMA/DSMEM, exactly
// pruned).  This file holds the plain unpruned scan (every element's Philox +
// noise evaluated, one CTA per row) — the product path for row shapes the
// cluster kernel does not take (V*esz not a multiple of 16, or an unaligned
// logits pointer) and the bit-exact reference the tests compare the pruned
// scan against (srt_sample_rows_reference) — and the accept/commit kernel.
#include <cuda_bf16.h>

#include "noise.cuh"
#include "srt_internal.cuh"
#include "accept.cuh"

namespace srt {

namespace {

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

__device__ __forceinline__ float load_elem(const void* row, int dtype, int64_t v) {
  if (dtype == SRT_BF16) {
    const uint16_t h = ((const uint16_t*)row)[v];
    return __uint_as_float((uint32_t)h << 16);
  }
  return ((const float*)row)[v];
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
// Writes sampled[r] directly, or (result != nullptr) the row's packed best
// candidate for the accept kernel (the product scan's output format).
__global__ void __launch_bounds__(REF_THREADS)
k_scan_reference(DevCache c, VerifyArgs a, unsigned long long* result) {
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
    // the definition, element by element (block constants recomputed per element)
    for (int64_t v = threadIdx.x; v < V; v += REF_THREADS) {
      const float x = load_elem(row, a.dtype, v);
      if (x != x) { nan_seen = true; continue; }
      const uint32_t b = (uint32_t)(v / NOISE_BLK), j = (uint32_t)(v % NOISE_BLK);
      const uint32_t n = (uint32_t)block_len(V, b);
      uint32_t wa, wb;
      block_words(b, (uint32_t)m.pos, m.sid_lo, m.sid_hi, k0, k1, wa, wb);
      const BlockNoise bn = block_noise(wa, wb, n);
      float g = bn.G;
      if (j != bn.p) {
        const Philox4 w = philox4x32_10((uint32_t)(v >> 2), (uint32_t)m.pos, m.sid_lo, m.sid_hi, k0, k1);
        const uint32_t k = (uint32_t)(v & 3);
        g = element_noise_from_word(k == 0 ? w.x : k == 1 ? w.y : k == 2 ? w.z : w.w, bn);
      }
      const float z = perturbed(x, g, a.temperature, unit_t);
      if (cand_better(z, (int32_t)v, bz, bv)) { bz = z; bv = (int32_t)v; }
    }
    if (nan_seen) set_error(c, SRT_DEV_NONFINITE_LOGIT);
    block_argmax<REF_THREADS>(bz, bv, sz, sv);
    if (threadIdx.x == 0) {
      if (result) result[r] = bv == INT_MAX ? 0ull : pack_cand(bz, bv);
      else a.sampled[r] = bv == INT_MAX ? 0 : bv;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Accept + commit: one warp per sequence.
// ---------------------------------------------------------------------------
constexpr int ACC_WARPS = 4;

// One warp per sequence (accept.cuh).
__global__ void __launch_bounds__(ACC_WARPS * 32)
k_accept(DevCache c, VerifyArgs a, const unsigned long long* __restrict__ result) {
  __shared__ int32_t ctok[ACC_WARPS][65];
  __shared__ int32_t acc[ACC_WARPS][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t s = blockIdx.x * ACC_WARPS + w;
  if (s >= a.n) return;
  accept_seq(c, a, result, s, ctok[w], acc[w], lane);
}

}  // namespace

cudaError_t launch_scan(const DevCache& c, const VerifyArgs& a, bool reference, int2* rowinfo,
                        unsigned long long* result, cudaStream_t stream) {
  const int C = scan_cluster_size(c.V, a.dtype);
  const bool aligned = ((uintptr_t)a.logits % 16) == 0;
  if (reference || C == 0 || !aligned || !result) {
    k_scan_reference<<<num_sms() * 8, REF_THREADS, 0, stream>>>(c, a, reference ? nullptr : result);
    return cudaGetLastError();
  }
  return launch_scan_cluster(c, a, rowinfo, result, stream);
}

cudaError_t launch_accept(const DevCache& c, const VerifyArgs& a, const unsigned long long* result,
                          cudaStream_t stream) {
  carveout_once<k_accept>();
  k_accept<<<(a.n + ACC_WARPS - 1) / ACC_WARPS, ACC_WARPS * 32, 0, stream>>>(c, a, result);
  return cudaGetLastError();
}

}  // namespace srt
