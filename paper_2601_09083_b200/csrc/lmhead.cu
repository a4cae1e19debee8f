// lmhead.cu — the verification pass without materialised logits (SURVEY
// §8(f3a)): the LM-head GEMM logits = hidden · W^T on the 5th-generation tensor
// cores with the exact Gumbel-max sampler of srt_verify (reading O11) as its
// epilogue, so the [rows, V] logits never reach HBM.  P:L139 ("one decode
// pass ... verify multiple drafted tokens in parallel"), P:L379 (decoding is
// memory-bandwidth bound: the 2 x rows x V x 2 B logits write + read is the
// traffic this removes).
//
// Persistent, warp-specialised, one CTA per SM:
//  * warp 0, one lane: TMA producer — 2-D tensor-map loads (128-byte swizzle)
//    of a 128 x 64 hidden tile and a 256 x 64 weight tile per K step into an
//    NST-stage shared-memory ring (mbarrier full/empty pairs);
//  * warp 1, one lane: tcgen05.mma issuer — 4 x (M128 N256 K16) bf16 MMAs per
//    stage into an fp32 accumulator in tensor memory (two 256-column
//    accumulators: the epilogue of tile i overlaps the MMAs of tile i + 1);
//    tcgen05.commit frees the stage / publishes the accumulator;
//  * warps 2-17: epilogue — tcgen05.ld of the thread's row (32x32b: thread =
//    TMEM lane = logits row; four warps per lane quarter, one per noise block
//    of the tile; the accumulator is released as soon as it is in
//    registers), the logit's rounding to the cache's logits
//    dtype (bf16 RN-even, exactly what a bf16 LM head would store), then the
//    scan's exact branch and bound per 64-token noise block: block maximum,
//    bound U_b = RN(max/T) + (bucket bound of G_b), exact z only where a
//    block can still reach the row's best achieved z (shared across tiles of
//    the row through result[row], whose packed (z, v) IS an achieved z).
// Tile order is vocabulary-major (tile t: vocab tile t / num_m, row block
// t % num_m): the CTAs in flight share one weight tile (L2-resident) and a
// row's vocabulary tiles run one after another, so its bound only tightens.
// The result is the argmax of the plain definition over the rounded logits
// (ties to the smaller index): srt_verify on the dumped logits returns the
// same bits (tests/test_gpu_lmhead.py).
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "noise.cuh"
#include "srt_internal.cuh"

namespace srt {

namespace {

constexpr int BM = 128;             // rows per CTA (TMEM lanes); the CTA pair covers 256
constexpr int BN = 256;             // vocabulary columns per tile (UMMA N)
constexpr int BK = 64;              // K per stage: 64 bf16 = one 128-byte swizzle row
constexpr int UK = 16;              // K per tcgen05.mma (kind::f16)
constexpr int NST = 6;              // smem ring stages
constexpr int A_BYTES = BM * BK * 2;             // 16 KB: this CTA's 128 rows of hidden
constexpr int B_BYTES = (BN / 2) * BK * 2;       // 16 KB: this CTA's half of the weight tile
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 32 KB
constexpr int EPI_WARPS = 16;
constexpr int THREADS = (2 + EPI_WARPS) * 32;
constexpr int TMEM_COLS = 2 * BN;   // two accumulators
constexpr int BLK_PER_TILE = BN / NOISE_BLK;     // 4 noise blocks per tile
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;      // shared::cluster address -> CTA 0 of the pair

// ---- PTX: shared-memory addresses, mbarriers, TMA, tcgen05 ---------------
__device__ __forceinline__ uint32_t sm32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(sm32(b)),
      "r"(parity)
      : "memory");
}
// 2-SM TMA: the bytes land in THIS CTA's shared memory and are counted on
// CTA 0's barrier (the one the pair's MMA issuer waits on)
__device__ __forceinline__ void tma_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(sm32(dst)),
      "l"((uint64_t)map), "r"(sm32(bar) & PEER_MASK), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
// arrive on CTA 0's copy of `bar`
__device__ __forceinline__ void bar_arrive_leader(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(sm32(b) & PEER_MASK)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// the epilogue's wait: a try_wait with a suspend-time hint parks the warp
// until the phase completes instead of polling (16 polling warps would take
// issue slots from the producer / MMA warps)
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 20000;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(sm32(b)), "r"(parity)
        : "memory");
    if (done) return;
  }
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T over the CTA pair (M = 256: each CTA's A
// rows land in its own TMEM; B's N halves come from both CTAs), both
// K-major; issued by one thread of CTA 0
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` in BOTH CTAs of the pair once every tcgen05 op this thread
// issued so far completes
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(sm32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor of a K-major tile in the 128-byte swizzle
// layout TMA writes (rows of 128 B, 8-row groups 1024 B apart): start >> 4,
// leading byte offset 16 B (unused by swizzled K-major), stride byte offset
// 1024 B, version 1 (tcgen05), layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = 2 BM (pair)
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

__device__ __forceinline__ uint64_t ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // .x = a (low half)
  return *reinterpret_cast<const uint32_t*>(&h);
}

// the logit as the cache's logits dtype stores it (bf16: RN-even), in fp32
template <int DT>
__device__ __forceinline__ float as_logit(float acc) {
  if (DT == SRT_BF16) return __bfloat162float(__float2bfloat16_rn(acc));
  return acc;
}

// z of element v (offset k in its block) with the block's noise bn: RN(xs + g_v).
// Out of line: the exact pass calls it for the few elements that pass the
// prefilter, from a 64-way unrolled loop.
// Before the two logarithms, a bound: g_v = min(G_b, -log_det(RN(E_b + A_v)))
// <= min(G_b, g(r_v)) + (8 ulp of log_det's non-monotonicity, bounded by its
// <= 4 ulp error vs log, pinned exhaustively) <= min(G_b, gstd[r_v >> 13] +
// 2^-14), gstd = the bucket maxima of g(r); if even that cannot reach M the
// element is skipped (returns -inf).
__device__ __noinline__ float elem_z(float xs, int64_t v, int32_t k, BlockNoise bn, uint32_t pos,
                                     uint32_t slo, uint32_t shi, uint32_t k0, uint32_t k1,
                                     float M, const float* gstd) {
  float g = bn.G;
  if ((uint32_t)k != bn.p) {
    const Philox4 w = philox4x32_10((uint32_t)(v >> 2), pos, slo, shi, k0, k1);
    const uint32_t e = (uint32_t)(v & 3);
    const uint32_t wv = e == 0 ? w.x : e == 1 ? w.y : e == 2 ? w.z : w.w;
    const float gb = fminf(bn.G, gstd[wv >> 22] + 6.103515625e-05f);
    if (__fadd_rn(xs, gb) < M) return -INFINITY;
    g = element_noise_from_word(wv, bn);
  }
  return __fadd_rn(xs, g);
}

// A raw-accumulator threshold below which RN(RN(RN_logit(x)/T) + G) < M
// for certain: (M - G) T lowered by a margin covering the logit rounding
// (2^-8 relative), the division and the addition (a few ulp each).
__device__ __forceinline__ float prefilter_threshold(float M, float G, float T) {
  if (!(M > -INFINITY)) return -INFINITY;
  const float c = (M - G) * T;
  const float thr = c - (fabsf(c) * 0.0625f + fabsf(M) * 0.0625f * T + 1e-30f);
  return thr == thr && thr < INFINITY ? thr : -INFINITY;  // (overflow: no prefilter)
}

__device__ unsigned long long g_lm_stats[4];  // development (SRT_LMHEAD_DEBUG & 64)

struct LmParams {
  int32_t V;
  int32_t nk;                  // K steps (ceil(K / 64))
  const int64_t* total;        // -> row_offsets[n]
  const int2* rowinfo;         // per row: (sequence, position)
  const uint64_t* seq_id;
  uint64_t seed;
  float temperature;
  unsigned long long* result;  // per row: packed best (z, v), atomicMax
  void* dump;                  // nullable [rows, V] logits
  void* cand_x;                // [rows][cand_cap][64] deferred blocks' rounded logits
  int32_t* cand_b;             // [rows][cand_cap] their block indices
  float* cand_X;               // [rows][cand_cap] their maxima (rounded)
  int32_t* cand_n;             // [rows] deferred blocks (may exceed cand_cap: overflow)
  int32_t cand_cap;
  uint32_t debug;              // development: 1 = epilogue skips its work, 2 = no MMAs,
                               // 4 = bounds only (no exact pass)
};

template <int DT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
k_lmhead_sample(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                DevCache c, LmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles (same offsets in both CTAs)
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* ring = smem;                                        // [NST][A | B half]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NST * STAGE_BYTES);
  uint64_t* empty = full + NST;
  uint64_t* acc_full = empty + NST;   // [2]
  uint64_t* acc_empty = acc_full + 2; // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* tab = reinterpret_cast<float*>(tmem_slot + 4);              // [NOISE_BUCKETS]
  float* gstd = tab + NOISE_BUCKETS;                                 // [NOISE_BUCKETS]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t rank = blockIdx.x & 1;  // in the CTA pair (cluster of 2)
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t total = *p.total;
  const int32_t num_m = (int32_t)((total + 2 * BM - 1) / (2 * BM));  // 256-row pair blocks
  const int32_t num_n = (p.V + BN - 1) / BN;
  const int64_t tiles = (int64_t)num_m * num_n;

  for (int i = tid; i < NOISE_BUCKETS; i += blockDim.x) {
    tab[i] = c.gbound[i];
    gstd[i] = c.gbound[2 * NOISE_BUCKETS + 1 + i];
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      bar_init(&full[s], 1);   // (CTA 0's: the leader's expect_tx; both CTAs' bytes)
      bar_init(&empty[s], 1);  // the MMA commit, multicast to both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&acc_full[a], 1);
      bar_init(&acc_empty[a], 2 * EPI_WARPS);  // (CTA 0's: both CTAs' epilogue warps)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_b) : "memory");
  }
  if (wid == 1) {  // warp 1 of both CTAs allocates the pair's tensor memory
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     sm32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (wid == 0) {
    // ============ TMA producer (both CTAs: own A rows, own half of B) =======
    if (lane == 0) {
      uint64_t pol_a, pol_b;  // hidden rows are re-read for every vocab tile; W once per m
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_b));
      uint32_t it = 0;
      for (int64_t t = pair; t < tiles; t += npairs) {
        const int32_t nt = (int32_t)(t / num_m), mb = (int32_t)(t % num_m);
        for (int32_t kb = 0; kb < p.nk; ++kb, ++it) {
          const int s = (int)(it % NST);
          const uint32_t use = it / NST;
          if (use > 0) bar_wait(&empty[s], (use - 1) & 1);
          unsigned char* st = ring + s * STAGE_BYTES;
          if (rank == 0) bar_expect_tx(&full[s], 2 * STAGE_BYTES);
          tma_2d_pair(st, &map_a, &full[s], kb * BK, mb * 2 * BM + (int32_t)rank * BM, pol_a);
          tma_2d_pair(st + A_BYTES, &map_b, &full[s], kb * BK, nt * BN + (int32_t)rank * (BN / 2),
                      pol_b);
        }
      }
    }
  } else if (wid == 1) {
    // ============ MMA issuer (CTA 0 only) =================================
    if (rank == 0) {
      uint32_t it = 0, u = 0;
      for (int64_t t = pair; t < tiles; t += npairs, ++u) {
        const uint32_t a = u & 1, ause = u >> 1;
        if (ause > 0) bar_wait(&acc_empty[a], (ause - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + a * BN;
        for (int32_t kb = 0; kb < p.nk; ++kb, ++it) {
          const int s = (int)(it % NST);
          bar_wait(&full[s], (it / NST) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = sm32(ring + s * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UK; ++k)  // +32 bytes per K16 step inside the swizzle row
              if (!(p.debug & 2))
                tc_mma(d, sw128_desc(sa + k * UK * 2), sw128_desc(sb + k * UK * 2), IDESC,
                       (kb | k) != 0);
            tc_commit(&empty[s]);                         // stage free in both CTAs
            if (kb == p.nk - 1) tc_commit(&acc_full[a]);  // accumulator complete in both
          }
          __syncwarp();
        }
      }
    }
  } else {
#ifdef SRT_LMHEAD_PROF
    long long tph[6] = {0, 0, 0, 0, 0, 0};
    const long long tp0 = clock64();
#define LMP(i, t) tph[i] += clock64() - (t)
#else
#define LMP(i, t) (void)0
#endif
    // ============ epilogue: sample from the accumulator ===================
    // 16 warps: warp w reads TMEM lanes 32 (w % 4) .. + 31 (its 32 rows) and
    // noise block jb = (w - 2) / 4 of the tile's four (columns 64 jb .. + 63).
    const int q = wid & 3;
    const int jb = (wid - 2) >> 2;
    const float T = p.temperature;
    const bool unit_t = T == 1.0f;
    const uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
    const int64_t nblk = ((int64_t)p.V + NOISE_BLK - 1) / NOISE_BLK;
    uint32_t u = 0;
    for (int64_t t = pair; t < tiles; t += npairs, ++u) {
      const uint32_t a = u & 1;
      const int32_t nt = (int32_t)(t / num_m), mb = (int32_t)(t % num_m);
      const int64_t r = (int64_t)mb * 2 * BM + rank * BM + q * 32 + lane;
      const bool rv = r < total;
      const int64_t b = (int64_t)nt * BLK_PER_TILE + jb;  // this warp's noise block
      const int n = block_len(p.V, b);
      // the row's key and best-so-far (global loads) before the accumulator wait
      long long tq = clock64();
      int2 ri = make_int2(0, 0);
      if (rv && !(p.debug & 8)) ri = p.rowinfo[r];
      uint32_t pos = 0, slo = 0, shi = 0;
      unsigned long long cur = 0;
      if (rv && !(p.debug & 8)) {
        const uint64_t sid = p.seq_id[ri.x];
        pos = (uint32_t)ri.y;
        slo = (uint32_t)sid;
        shi = (uint32_t)(sid >> 32);
        cur = ld_relaxed64(&p.result[r]);
      }
      uint32_t wa = 0, wb = 0;  // the block's words (one Philox call per block pair)
      if (rv && b < nblk) {
        const Philox4 w = philox4x32_10(0x80000000u | (uint32_t)(b >> 1), pos, slo, shi, k0, k1);
        wa = (b & 1) ? w.z : w.x;
        wb = (b & 1) ? w.w : w.y;
      }
      LMP(0, tq);
      tq = clock64();
      bar_wait_sleep(&acc_full[a], (u >> 1) & 1);
      tc_fence_after();
      LMP(1, tq);
      tq = clock64();
      if (p.debug & 1) {  // development: the pipeline without the sampler
        __syncwarp();
        if (lane == 0) bar_arrive_leader(&acc_empty[a]);
        continue;
      }
      float x[NOISE_BLK];
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + a * BN + jb * NOISE_BLK;
      tmem_ld32(taddr, x);
      tmem_ld32(taddr + 32, x + 32);
      // the accumulator stays in registers: release it to the MMA right away
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive_leader(&acc_empty[a]);
      LMP(2, tq);
      tq = clock64();
      // ---- the block maximum X: rounding is monotone, so the max of the
      // rounded logits is the rounded max of the accumulators ----
      bool nan = false;
      float m = -INFINITY;
      if (n == NOISE_BLK) {
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int k = 0; k < NOISE_BLK; k += 2) {
          m0 = max_nan(m0, x[k]);
          m1 = max_nan(m1, x[k + 1]);
        }
        m = max_nan(m0, m1);
      }
      if (n < NOISE_BLK || m != m) {  // partial block, or a NaN: the careful max
        m = -INFINITY;
#pragma unroll
        for (int k = 0; k < NOISE_BLK; ++k)
          if (k < n) {
            nan |= x[k] != x[k];
            if (x[k] > m) m = x[k];
          }
      }
      const float X = n > 0 ? as_logit<DT>(m) : -INFINITY;
      if (p.dump && rv && n > 0) {
        const int64_t v0 = b * NOISE_BLK;
        if (DT == SRT_BF16) {
          __nv_bfloat16* o = (__nv_bfloat16*)p.dump + r * (int64_t)p.V + v0;
#pragma unroll
          for (int k = 0; k < NOISE_BLK; ++k)
            if (k < n) o[k] = __float2bfloat16_rn(x[k]);
        } else {
          float* o = (float*)p.dump + r * (int64_t)p.V + v0;
#pragma unroll
          for (int k = 0; k < NOISE_BLK; ++k)
            if (k < n) o[k] = x[k];
        }
      }
      float M = cur ? unpack_value(cur) : -INFINITY;  // an achieved z of the row (or none)
      float bz = -INFINITY;
      int32_t bv = INT_MAX;
      const float Xs = unit_t ? X : __fdiv_rn(X, T);
      float U = -INFINITY;  // the block bound RN(X/T) + (bucket bound of G_b)
      if (rv && n > 0 && X > -INFINITY)
        U = __fadd_rn(Xs, n == NOISE_BLK ? tab[wa >> 22] : block_noise(wa, wb, (uint32_t)n).G);
      if (p.debug & 32) U = -INFINITY;
      if (p.debug & 64) {
        const unsigned nb = __popc(__ballot_sync(0xffffffffu, U > -INFINITY && U >= M));
        const unsigned nw = __any_sync(0xffffffffu, U > -INFINITY && U >= M);
        if (lane == 0) {
          atomicAdd(&g_lm_stats[0], nb);   // lane-blocks evaluated
          atomicAdd(&g_lm_stats[1], nw);   // warp-blocks with any evaluation
          atomicAdd(&g_lm_stats[3], 1ull); // warp-blocks
        }
      }
      LMP(3, tq);
      tq = clock64();
      if (U > -INFINITY && U >= M && !(p.debug & 16)) {
        // ---- the block can still hold the row's winner ----
        const BlockNoise bn = block_noise(wa, wb, (uint32_t)n);
        const int64_t vb = b * NOISE_BLK;
        // z(i*) of an element holding the block maximum (raw max m: its
        // rounded value is X): an achieved z, which raises the row's bound for
        // every later tile
        int32_t ks = 0;
#pragma unroll
        for (int k = NOISE_BLK - 1; k >= 0; --k)
          if (k < n && x[k] == m) ks = k;
        const float zs = elem_z(Xs, vb + ks, ks, bn, pos, slo, shi, k0, k1, -INFINITY, gstd);
        bz = zs;
        bv = (int32_t)(vb + ks);
        M = fmaxf(M, zs);
        // can any other element still reach M?  (RN(RN(x/T) + G_b) >= M, a
        // raw-value prefilter first)
        const float thr = prefilter_threshold(M, bn.G, T);
        bool open = false;
#pragma unroll
        for (int k = 0; k < NOISE_BLK; ++k) {
          if (k < n && k != ks && x[k] >= thr) {
            const float xr = as_logit<DT>(x[k]);
            const float xs = unit_t ? xr : __fdiv_rn(xr, T);
            open |= __fadd_rn(xs, bn.G) >= M;
          }
        }
        if (p.debug & 64) atomicAdd(&g_lm_stats[2], (unsigned long long)open);
        if (open) {
          // defer the block: its rounded logits go to the row's candidate
          // list, evaluated exactly by k_lmhead_tail against the row's final
          // bound; a full list falls back to an inline exact pass
          const int32_t slot = atomicAdd(&p.cand_n[r], 1);
          if (slot < p.cand_cap) {
            const int64_t e = r * (int64_t)p.cand_cap + slot;
            p.cand_b[e] = (int32_t)b;
            p.cand_X[e] = X;
            if (DT == SRT_BF16) {
              uint4* o = reinterpret_cast<uint4*>((__nv_bfloat16*)p.cand_x + e * NOISE_BLK);
#pragma unroll
              for (int k = 0; k < NOISE_BLK; k += 8) {
                uint4 w;
                w.x = pack_bf2(x[k], x[k + 1]);
                w.y = pack_bf2(x[k + 2], x[k + 3]);
                w.z = pack_bf2(x[k + 4], x[k + 5]);
                w.w = pack_bf2(x[k + 6], x[k + 7]);
                o[k / 8] = w;
              }
            } else {
              float4* o = reinterpret_cast<float4*>((float*)p.cand_x + e * NOISE_BLK);
#pragma unroll
              for (int k = 0; k < NOISE_BLK; k += 4)
                o[k / 4] = make_float4(x[k], x[k + 1], x[k + 2], x[k + 3]);
            }
          } else {
#pragma unroll 1
            for (int k = 0; k < n; ++k) {  // overflow: every element, inline
              float xk = 0.0f;
#pragma unroll
              for (int i = 0; i < NOISE_BLK; ++i)
                if (i == k) xk = x[i];
              const float xr = as_logit<DT>(xk);
              const float xs = unit_t ? xr : __fdiv_rn(xr, T);
              if (k == ks || __fadd_rn(xs, bn.G) < M) continue;
              const float z = elem_z(xs, vb + k, k, bn, pos, slo, shi, k0, k1, M, gstd);
              if (cand_better(z, (int32_t)(vb + k), bz, bv)) {
                bz = z;
                bv = (int32_t)(vb + k);
                M = fmaxf(M, z);
              }
            }
          }
        }
      }
      LMP(4, tq);
      tq = clock64();
      if (__any_sync(0xffffffffu, nan) && lane == 0) set_error(c, SRT_DEV_NONFINITE_LOGIT);
      if (rv && bv != INT_MAX) {
        const unsigned long long pk = pack_cand(bz, bv);
        if (pk > cur) atomicMax(&p.result[r], pk);
      }
      LMP(5, tq);
    }
#ifdef SRT_LMHEAD_PROF
    if (blockIdx.x < 2 && lane == 0)
      printf("[lm prof] cta %d warp %2d total %lld loads %lld wait %lld tmem %lld bound %lld exact %lld out %lld tiles %u\n",
             blockIdx.x, wid, clock64() - tp0, tph[0], tph[1], tph[2], tph[3], tph[4], tph[5], u);
#endif
#undef LMP
  }
  tc_fence_before();
  cluster_sync();  // both CTAs done with the tensor memory and the leader's barriers
  if (wid == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// The deferred blocks of each row, exactly, against the row's final bound M
// (the best achieved z over all its tiles -- in practice the head's): one
// warp per row, two tokens per lane per block.  Every block the GEMM
// epilogue pruned had U_b < M at the time, and M only grew, so the argmax
// over the deferred blocks and the epilogue's candidates is the row's.
template <int DT>
__global__ void __launch_bounds__(128) k_lmhead_tail(DevCache c, LmParams p) {
  __shared__ float tab[NOISE_BUCKETS];
  for (int i = threadIdx.x; i < NOISE_BUCKETS; i += blockDim.x) tab[i] = c.gbound[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t total = *p.total;
  const float T = p.temperature;
  const bool unit_t = T == 1.0f;
  const uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
  const float* gstd = c.gbound + 2 * NOISE_BUCKETS + 1;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < total;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t nd = p.cand_n[r];
    if (nd == 0) continue;
    const int32_t nc = min(nd, p.cand_cap);
    const unsigned long long cur = ld_relaxed64(&p.result[r]);
    float M = cur ? unpack_value(cur) : -INFINITY;
    const int2 ri = p.rowinfo[r];
    const uint64_t sid = p.seq_id[ri.x];
    const uint32_t pos = (uint32_t)ri.y, slo = (uint32_t)sid, shi = (uint32_t)(sid >> 32);
    float bz = -INFINITY;
    int32_t bv = INT_MAX;
    for (int32_t i0 = 0; i0 < nc; i0 += 32) {
      // lane i: deferred block i0 + i -- its bound against the row's final M
      const int32_t i = i0 + lane;
      const int64_t e = r * (int64_t)p.cand_cap + i;
      int64_t b = 0;
      float U = -INFINITY;
      if (i < nc) {
        b = p.cand_b[e];
        const float X = p.cand_X[e];
        const int n = block_len(p.V, b);
        uint32_t wa, wb;
        block_words((uint32_t)b, pos, slo, shi, k0, k1, wa, wb);
        const float G = n == NOISE_BLK ? tab[wa >> 22] : block_noise(wa, wb, (uint32_t)n).G;
        U = __fadd_rn(unit_t ? X : __fdiv_rn(X, T), G);
      }
      unsigned surv = __ballot_sync(0xffffffffu, U > -INFINITY && U >= M);
      while (surv) {  // the surviving blocks, exactly, by the whole warp
        const int j = __ffs(surv) - 1;
        surv &= surv - 1;
        const int64_t bj = __shfl_sync(0xffffffffu, b, j);
        const int64_t ej = r * (int64_t)p.cand_cap + i0 + j;
        const int n = block_len(p.V, bj);
        uint32_t wa, wb;
        block_words((uint32_t)bj, pos, slo, shi, k0, k1, wa, wb);
        const BlockNoise bn = block_noise(wa, wb, (uint32_t)n);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 2 * lane + h;
          if (k >= n) continue;
          const float x = DT == SRT_BF16
                              ? __bfloat162float(((const __nv_bfloat16*)p.cand_x)[ej * NOISE_BLK + k])
                              : ((const float*)p.cand_x)[ej * NOISE_BLK + k];
          const float xs = unit_t ? x : __fdiv_rn(x, T);
          if (!(__fadd_rn(xs, bn.G) >= M)) continue;
          const int64_t v = bj * NOISE_BLK + k;
          const float z = elem_z(xs, v, k, bn, pos, slo, shi, k0, k1, M, gstd);
          if (cand_better(z, (int32_t)v, bz, bv)) {
            bz = z;
            bv = (int32_t)v;
          }
        }
        // the warp's best z tightens the bound for the remaining blocks
        float wm = bz;
        for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        M = fmaxf(M, wm);
        surv &= __ballot_sync(0xffffffffu, U > -INFINITY && U >= M);
      }
    }
    // the warp's best (larger z, then smaller v) -> the row's packed result
    const unsigned long long mine = bv == INT_MAX ? 0ull : pack_cand(bz, bv);
    const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(mine >> 32));
    const uint32_t lo =
        __reduce_max_sync(0xffffffffu, (uint32_t)(mine >> 32) == hi ? (uint32_t)mine : 0u);
    const unsigned long long best = ((unsigned long long)hi << 32) | lo;
    if (lane == 0) {
      if (best > cur) atomicMax(&p.result[r], best);
      p.cand_n[r] = 0;  // (clean for the next call)
    }
  }
}


// A lower bound on each row's winning z before the GEMM (§8d): the row's
// first drafted child token (the draft's most likely continuation; none for
// a leaf row) gets its logit as a CUDA-core fp32 dot product, lowered by a
// margin that covers both that sum's and the tensor cores' accumulation
// error (2 K 2^-20 sum |h_k w_k|: 16x the fp32 bound), rounded like the
// kernel's logit (monotone, so still below the logit the kernel will see),
// and z = RN(RN(x/T) + g) with the element's exact noise (O11).  That is a
// lower bound on an achieved z of the row, so every block whose bound is
// below it can be skipped from the first tile on; it is stored as the row's
// packed candidate (hint's exact z >= it replaces it when the hint's block is
// evaluated, and any winner beats it), never returned as such unless exact.
template <int DT>
__global__ void __launch_bounds__(256) k_lmhead_seed(DevCache c, VerifyArgs a,
                                                     const __nv_bfloat16* __restrict__ hidden,
                                                     const __nv_bfloat16* __restrict__ W, int32_t K,
                                                     const int2* __restrict__ rowinfo,
                                                     unsigned long long* __restrict__ result) {
  const int lane = threadIdx.x & 31;
  const int64_t total = a.row_offsets[a.n];
  const int32_t B = c.Bmax;
  const float T = a.temperature;
  const bool unit_t = T == 1.0f;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < total;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int2 ri = rowinfo[r];
    const int32_t s = ri.x;
    const int32_t i = (int32_t)(r - a.row_offsets[s]);  // 0 = root row, else node i - 1
    const int32_t nd = a.draft_len[s];
    const int32_t* par = a.draft_parent + (int64_t)s * B;
    // the node's first child in pop order (children follow their parent)
    const bool ca = lane < nd && lane >= i && par[lane] == i - 1;
    const bool cb = lane + 32 < nd && lane + 32 >= i && par[lane + 32] == i - 1;
    const unsigned ma = __ballot_sync(0xffffffffu, ca), mb = __ballot_sync(0xffffffffu, cb);
    if (!(ma | mb)) continue;
    const int32_t j = ma ? __ffs(ma) - 1 : 31 + __ffs(mb);
    const int32_t hint = a.draft_tok[(int64_t)s * B + j];
    if (hint < 0 || hint >= c.V) continue;
    const __nv_bfloat16* h = hidden + r * (int64_t)K;
    const __nv_bfloat16* w = W + (int64_t)hint * K;
    float d = 0.0f, sabs = 0.0f;
    for (int32_t k = lane * 8; k < K; k += 256) {  // K % 8 == 0 (checked on the host)
      const uint4 hv = *reinterpret_cast<const uint4*>(h + k);
      const uint4 wv = *reinterpret_cast<const uint4*>(w + k);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hv);
      const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wv);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 hf = __bfloat1622float2(h2[q]), wf = __bfloat1622float2(w2[q]);
        d = fmaf(hf.x, wf.x, d);
        d = fmaf(hf.y, wf.y, d);
        sabs += fabsf(hf.x * wf.x) + fabsf(hf.y * wf.y);
      }
    }
    for (int o = 16; o; o >>= 1) {
      d += __shfl_xor_sync(0xffffffffu, d, o);
      sabs += __shfl_xor_sync(0xffffffffu, sabs, o);
    }
    const float margin = 2.0f * (float)K * 9.5367431640625e-07f * sabs * 1.0001f;  // 2^-20
    const float x = as_logit<DT>(d - margin);
    if (!(x > -INFINITY) || !(x < INFINITY)) continue;
    // the hint element's noise (O11)
    const int64_t b = hint / NOISE_BLK;
    const int n = block_len(c.V, b);
    uint32_t wa, wb;
    block_words((uint32_t)b, (uint32_t)ri.y, (uint32_t)a.seq_id[s], (uint32_t)(a.seq_id[s] >> 32),
                k0, k1, wa, wb);
    const BlockNoise bn = block_noise(wa, wb, (uint32_t)n);
    float g = bn.G;
    const uint32_t jb = (uint32_t)(hint - b * NOISE_BLK);
    if (jb != bn.p) {
      const Philox4 pw = philox4x32_10((uint32_t)(hint >> 2), (uint32_t)ri.y,
                                       (uint32_t)a.seq_id[s], (uint32_t)(a.seq_id[s] >> 32), k0, k1);
      const uint32_t e = (uint32_t)(hint & 3);
      g = element_noise_from_word(e == 0 ? pw.x : e == 1 ? pw.y : e == 2 ? pw.z : pw.w, bn);
    }
    const float z = perturbed(x, g, T, unit_t);
    if (lane == 0 && z == z) atomicMax(&result[r], pack_cand(z, hint));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows, K] matrix, box [box_rows, 64],
// 128-byte swizzle (the UMMA K-major SW128 layout); out-of-range reads are 0
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int32_t K, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_lmhead_sample(const DevCache& c, const VerifyArgs& a, const LmHeadArgs& h,
                                 const int2* rowinfo, unsigned long long* result,
                                 const LmHeadScratch& sc, cudaStream_t stream) {
  CUtensorMap ma, mb;
  if (!make_map(&ma, h.hidden, h.hidden_rows, h.K, BM) ||
      !make_map(&mb, h.weight, c.V, h.K, BN / 2))
    return cudaErrorInvalidValue;
  LmParams p;
  p.V = c.V;
  p.nk = (h.K + BK - 1) / BK;
  p.total = a.row_offsets + a.n;
  p.rowinfo = rowinfo;
  p.seq_id = a.seq_id;
  p.seed = a.seed;
  p.temperature = a.temperature;
  p.result = result;
  p.dump = h.dump;
  p.cand_x = sc.cand_x;
  p.cand_b = sc.cand_b;
  p.cand_X = sc.cand_X;
  p.cand_n = sc.cand_n;
  p.cand_cap = sc.cap;
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = getenv("SRT_LMHEAD_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  p.debug = (uint32_t)dbg;
  const size_t smem = 1024 + (size_t)NST * STAGE_BYTES + 2 * NST * 8 + 4 * 8 + 16 +
                      2 * NOISE_BUCKETS * 4;
  auto kern = a.dtype == SRT_BF16 ? k_lmhead_sample<SRT_BF16> : k_lmhead_sample<SRT_F32>;
  if (!(p.debug & 256)) {  // the rows' seeded bounds (debug 256: off)
    auto sk = a.dtype == SRT_BF16 ? k_lmhead_seed<SRT_BF16> : k_lmhead_seed<SRT_F32>;
    sk<<<num_sms() * 8, 256, 0, stream>>>(c, a, (const __nv_bfloat16*)h.hidden,
                                          (const __nv_bfloat16*)h.weight, h.K, rowinfo, result);
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p.debug & 64) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbolAsync(g_lm_stats, z, sizeof z, 0, cudaMemcpyHostToDevice, stream);
  }
  kern<<<num_sms() & ~1, THREADS, smem, stream>>>(ma, mb, c, p);  // CTA pairs (cluster of 2)
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.debug & 128) {
  } else if (a.dtype == SRT_BF16)
    k_lmhead_tail<SRT_BF16><<<num_sms() * 8, 128, 0, stream>>>(c, p);
  else
    k_lmhead_tail<SRT_F32><<<num_sms() * 8, 128, 0, stream>>>(c, p);
  if (p.debug & 64) {
    unsigned long long z[4];
    cudaMemcpyFromSymbolAsync(z, g_lm_stats, sizeof z, 0, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    fprintf(stderr, "[lmhead] lane-blocks evaluated %llu, warp-blocks with work %llu of %llu, "
            "elements evaluated %llu\n", z[0], z[1], z[3], z[2]);
  }
  return cudaGetLastError();
}

}  // namespace srt
