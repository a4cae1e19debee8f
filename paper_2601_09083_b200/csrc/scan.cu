// scan.cu — the roofline kernel of srt_verify: the exact Gumbel-max sample of
// every drafted logits row (BJ:north_star part 4; O11 and §5).
//
// The noise is the top-down construction of O11: per block of 64 tokens the
// block's MAXIMUM noise G_b is drawn first (one Philox call per two blocks),
// the other 63 are Gumbels truncated below it.  So
//     U_b = RN(RN(max_{v in b} x_v / T) + G_b)  >=  z_v  for every v in b,
// and with the bucket bound G_b <= TAB[r_b >> 13] (the max of G over the
// block word's bucket, enumerated over all 2^23 words at cache creation) the
// block bound needs no logarithm at all.  A block can hold the row's winner
// only if U_b >= M for M any ACHIEVED z of the row; M = z(i*) of the row's
// largest logit is exact and strong.  Everything else is streaming.
//
// Persistent, warp-specialised kernel; one CTA per SM owns whole rows
// (rows b, b+G, b+2G, ...), so no row ever waits on another SM:
//  * producer warp: 1-D TMA bulk copies (cp.async.bulk + mbarrier) stream each
//    row through a ring of NST 32 KB shared-memory stages (~7.4 TB/s
//    read-only on this B200 in isolation, tools/stream_probe.cu);
//  * stream warps: each lane takes a PAIR of blocks (128 logits) per step —
//    packed bf16x2 maxima from conflict-free swizzled 16-byte shared loads,
//    one Philox call for the pair, the bucket-bounded U_b into the row summary
//    (4 B per block), and the row's largest logit;
//  * tail warps, one row behind: M = z(i*) exactly, then every block with
//    U_b >= M (the head's block and a few others) is evaluated element by
//    element from L2 with the exact noise; each warp's best (z, v) goes to the
//    row's packed atomicMax word (larger z, then smaller v).
// Nothing observable depends on scheduling: the result is the argmax of the
// plain definition (k_scan_reference; the tests compare both bit for bit).
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>

#include "noise.cuh"
#include "srt_internal.cuh"

#ifdef SRT_SCAN_PROF
#define SRT_SCAN_PROF_ON 1
#else
#define SRT_SCAN_PROF_ON 0
#endif

namespace srt {

namespace {

// ---- PTX helpers: mbarriers, 1-D TMA bulk copy ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  // (a suspend-time hint of ~10 ms was measured 0.5 % slower on the scan)
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// non-suspending variant: poll with test_wait (a try_wait may park the warp
// for a scheduler time slice after the phase completes)
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SPIN_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SPIN_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// same, with an L2 cache-policy hint (a development knob since r02 v5: no
// policy on the streamed rows measured fastest in the step)
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ __nv_bfloat162 as_bf2(uint32_t w) {
  return *reinterpret_cast<const __nv_bfloat162*>(&w);
}
// order-preserving key of a non-NaN float (never 0, which means "none")
__device__ __forceinline__ uint32_t fkey(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_value(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// block_len for V < 2^31 in 32-bit arithmetic (the hot loops)
__device__ __forceinline__ int block_len32(int32_t V, int32_t b) {
  const int32_t rem = V - b * NOISE_BLK;
  return rem <= 0 ? 0 : (rem < NOISE_BLK ? rem : NOISE_BLK);
}

template <int DT>
__device__ __forceinline__ float load_x(const unsigned char* rowp, int64_t v) {
  if (DT == SRT_BF16) return __uint_as_float((uint32_t)((const uint16_t*)rowp)[v] << 16);
  return ((const float*)rowp)[v];
}

// NaN-propagating max of the 16-byte vectors of one block held in shared
// memory: vector index (k + rot) & (NV - 1) at step k, so the 8 lanes of an
// LDS.128 phase hit distinct bank groups.
template <int DT>
__device__ __forceinline__ float block_max_nan(const unsigned char* blk, int rot) {
  constexpr int NV = DT == SRT_BF16 ? 8 : 16;  // 16-byte vectors per 64-token block
  const uint4* v = reinterpret_cast<const uint4*>(blk);
  if (DT == SRT_BF16) {
    __nv_bfloat162 m0 = as_bf2(0xFF80FF80u), m1 = m0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const uint4 q = v[(k + rot) & (NV - 1)];
      m0 = __hmax2_nan(m0, __hmax2_nan(as_bf2(q.x), as_bf2(q.y)));
      m1 = __hmax2_nan(m1, __hmax2_nan(as_bf2(q.z), as_bf2(q.w)));
    }
    const __nv_bfloat162 m = __hmax2_nan(m0, m1);
    return max_nan(__low2float(m), __high2float(m));
  } else {
    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const uint4 q = v[(k + rot) & (NV - 1)];
      m0 = max_nan(m0, max_nan(__uint_as_float(q.x), __uint_as_float(q.y)));
      m1 = max_nan(m1, max_nan(__uint_as_float(q.z), __uint_as_float(q.w)));
    }
    return max_nan(m0, m1);
  }
}

// non-NaN max of the first n elements of a block in shared memory (-inf if none)
template <int DT>
__device__ __forceinline__ float block_max_scalar(const unsigned char* blk, int n) {
  float m = -INFINITY;
  for (int j = 0; j < n; ++j) {
    const float x = load_x<DT>(blk, j);
    if (x > m) m = x;
  }
  return m;
}


struct ScanParams {
  const void* logits;
  const int2* rowinfo;         // per row: (seq, pos)
  const int32_t* row_list;     // nullable: scan rows row_list[0 .. total) instead of [0, total)
  const int64_t* total;        // -> row_offsets[n]
  const uint64_t* seq_id;
  uint64_t seed;
  float temperature;
  unsigned long long* result;  // per row: packed best candidate (atomicMax)
  int32_t V;
  int32_t nblk;                // ceil(V / 64)
  uint32_t sum_bytes;          // row summary bytes (nblk floats, 128-aligned)
  uint32_t debug;              // development only (SRT_SCAN_DEBUG: 8 prints the launch; 16 / 32
                               // skip the tail / stream work, timing probes with wrong results;
                               // 64: CTA 0 prints per-warp wait cycles)
  uint32_t l2_hint;            // 0 = no policy (default); 1-4 = development modes (below)
  uint32_t spin;               // 1 = stream warps poll the ring with test_wait
  uint32_t* sched;             // nullable: [0] next row to claim, [1] CTAs past the end (both 0
                               // between launches); null = static rows blockIdx.x + k gridDim.x
  uint32_t* seq_done;          // nullable: per sequence, rows whose result is final (the last
                               // worker of a row counts it, after its fence: the fused tree
                               // step beside the scan waits on these)
  int grid_cap;                // host side: at most this many CTAs (0 = one per SM)
};

// Warp roles: warp 0 = producer, warps 1..NSW = stream (NG groups taking
// alternate chunks, so NG chunks are summarised at once), the rest = tail.
template <int DT, int NSW, int NT, int NST, int NS, uint32_t CHUNK, int NG>
__global__ void __launch_bounds__((1 + NSW + NT) * 32, 1) k_scan_rows(DevCache c, ScanParams a) {
  constexpr int GW = NSW / NG;  // warps per stream group
  static_assert(NSW % NG == 0, "stream groups must be equal");
  static_assert(NT >= 2, "the tail needs the M warp and at least one worker");
  // each ring stage must always be consumed by the same group, in order: a
  // parity wait cannot tell use k from use k + 2
  static_assert(NST % NG == 0, "ring stages must map to one stream group each");
  constexpr int ESZ = DT == SRT_BF16 ? 2 : 4;
  constexpr int BLKB = NOISE_BLK * ESZ;  // bytes per block
  constexpr int PAIRB = 2 * BLKB;
  constexpr int PAIRS_PER_CHUNK = CHUNK / PAIRB;
  constexpr int NR = NST + 2;  // row ids the producer may run ahead by (see the stream loop)
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                            // [NST][CHUNK]
  unsigned char* sums = ring + NST * CHUNK;                              // [NS][sum_bytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sums + NS * a.sum_bytes);
  uint64_t* ring_full = bars;                                            // [NST]
  uint64_t* ring_empty = ring_full + NST;                                // [NST]
  uint64_t* sum_ready = ring_empty + NST;                                // [NS]
  uint64_t* sum_free = sum_ready + NS;                                   // [NS]
  uint64_t* m_ready = sum_free + NS;                                     // [NS]
  unsigned long long* p1key = reinterpret_cast<unsigned long long*>(m_ready + NS);  // [NS]
  unsigned long long* rowhdr = p1key + NS;                               // [NS]
  int64_t* rowid = reinterpret_cast<int64_t*>(rowhdr + NS);              // [NS] row of a summary
  int64_t* row_of = rowid + NS;                                          // [NR] row of the u-th row
  uint32_t* p1cnt = reinterpret_cast<uint32_t*>(row_of + NR);            // [NS]
  uint32_t* rowM = p1cnt + ((NS + 3) & ~3);                              // [NS] shared M keys
  float* tab = reinterpret_cast<float*>(rowM + ((NS + 3) & ~3));         // [1024]
  uint32_t* wdone = reinterpret_cast<uint32_t*>(tab + NOISE_BUCKETS);    // [NS] workers done
  // per row: (position, sequence id lo, hi, sequence), fetched by the
  // producer one row ahead (meta_p, like row_of) and handed to the tail with
  // the summary (meta_s): no warp on the stream's path waits on the two
  // dependent global loads (rowinfo, then seq_id) at a row's start
  uint4* meta_p = reinterpret_cast<uint4*>(wdone + ((NS + 3) & ~3));   // [NR]
  uint4* meta_s = meta_p + NR;                                           // [NS]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t total = *a.total;
  // (built with -DSRT_SCAN_PROF and debug 64: CTA 0's warps print the cycles
  // they spent in each wait; tools/build_ab.sh)
#ifdef SRT_SCAN_PROF
  const bool prof = (a.debug & 64) && blockIdx.x == 0;
#else
  constexpr bool prof = false;
#endif
  long long tw0 = 0, tw1 = 0, tw2 = 0, t_start = prof ? clock64() : 0;
  unsigned long long g_start = 0;
  if (SRT_SCAN_PROF_ON && (a.debug & 128)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
#define SRT_TIMED(acc, stmt)                     \
  do {                                           \
    if (prof) {                                  \
      const long long _t = clock64();            \
      stmt;                                      \
      acc += clock64() - _t;                     \
    } else {                                     \
      stmt;                                      \
    }                                            \
  } while (0)
#define SRT_PROF_PRINT(role)                                                                 \
  if (SRT_SCAN_PROF_ON && prof && lane == 0)                                                 \
    printf("[scan prof] warp %2d %-8s total %lld  w0 %lld  w1 %lld  w2 %lld\n", wid, role,   \
           clock64() - t_start, tw0, tw1, tw2)
  const int64_t row_bytes = (int64_t)a.V * ESZ;
  const uint32_t nch = (uint32_t)((row_bytes + CHUNK - 1) / CHUNK);
  const float T = a.temperature;
  const bool unit_t = T == 1.0f;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);

  for (int i = tid; i < NOISE_BUCKETS; i += blockDim.x) tab[i] = c.gbound[i];
  // the fused tree step beside the scan is this launch's programmatic
  // dependent: let it start now (it syncs on seq_done, not on completion)
  if (a.seq_done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&ring_full[s], 1);
      mbar_init(&ring_empty[s], GW);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sum_ready[s], 1);
      mbar_init(&sum_free[s], NT - 1);  // the workers
      mbar_init(&m_ready[s], 1);
      p1key[s] = 0;
      p1cnt[s] = 0;
      rowM[s] = 0;
      wdone[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == 0) {
    // ===================== producer: the rows' chunks into the ring ========
    if (lane == 0) {
      uint64_t pol = 0;
      // (development knob: 1 evict_first, 2 evict_first on half the lines,
      // 3 evict_unchanged, 4 evict_normal; 0 = no policy, the default)
      if (a.l2_hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else if (a.l2_hint == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 0.5;" : "=l"(pol));
      else if (a.l2_hint == 3) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
      else if (a.l2_hint == 4) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      // Rows are claimed one at a time from the launch's shared counter
      // (a.sched; else the static sequence blockIdx.x, + gridDim.x, ...), so
      // a CTA that met slow rows takes fewer of them.  The u-th row's id goes
      // to row_of[u % NR] before its first chunk is issued (the stream warps
      // read it after that chunk's full barrier); past the last row, one
      // empty arrival per stream group carries the end (row id -1).
      uint64_t kc = 0;
      int64_t si = blockIdx.x;
      auto claim = [&]() -> int64_t {
        if (a.sched) return (int64_t)atomicAdd(a.sched, 1u);
        const int64_t r = si;
        si += gridDim.x;
        return r;
      };
      // the row after the current one: claimed, and its meta fetched, while
      // the current row's first chunk is in flight (the ring's other stages
      // hide the round trips)
      auto fetch = [&](int64_t i, int64_t& row, uint4& m) {
        row = a.row_list ? a.row_list[i] : i;
        const int2 ri = a.rowinfo[row];
        const uint64_t sid = a.seq_id[ri.x];
        m = make_uint4((uint32_t)ri.y, (uint32_t)sid, (uint32_t)(sid >> 32), (uint32_t)ri.x);
      };
      int64_t next = claim();
      int64_t nrow = -1;
      uint4 nmeta = make_uint4(0, 0, 0, 0);
      if (next < total) fetch(next, nrow, nmeta);
      for (int64_t u = 0;; ++u) {
        const int64_t i = next;
        const int64_t row = nrow;
        const uint4 meta = nmeta;
        if (i < total) next = claim();
        if (i >= total) {
          row_of[u % NR] = -1;
          for (int g = 0; g < NG; ++g, ++kc) {
            const int s = (int)(kc % NST);
            const uint32_t use = (uint32_t)(kc / NST);
            if (use > 0) mbar_wait(&ring_empty[s], (use - 1) & 1);
            mbar_arrive(&ring_full[s]);
          }
          // the last CTA past the end resets the counter for the next launch
          if (a.sched && atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
            atomicExch(a.sched, 0u);
            atomicExch(a.sched + 1, 0u);
          }
          break;
        }
        row_of[u % NR] = row;
        meta_p[u % NR] = meta;
        const char* base = (const char*)a.logits + row * row_bytes;
        for (uint32_t ch = 0; ch < nch; ++ch, ++kc) {
          const int s = (int)(kc % NST);
          const uint32_t use = (uint32_t)(kc / NST);
          if (use > 0) {
            SRT_TIMED(tw0, mbar_wait(&ring_empty[s], (use - 1) & 1));
            // the stream warps' generic-proxy reads of the stage are ordered
            // before the async-proxy (TMA) overwrite
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
          const int64_t left = row_bytes - (int64_t)ch * CHUNK;
          const uint32_t nb = (uint32_t)(left < (int64_t)CHUNK ? left : (int64_t)CHUNK);
          mbar_arrive_expect_tx(&ring_full[s], nb);
          if (a.l2_hint)
            tma_load_1d_hint(ring + s * CHUNK, base + (int64_t)ch * CHUNK, nb, &ring_full[s], pol);
          else
            tma_load_1d(ring + s * CHUNK, base + (int64_t)ch * CHUNK, nb, &ring_full[s]);
          if (ch == 0 && next < total) fetch(next, nrow, nmeta);
        }
      }
      SRT_PROF_PRINT("producer");
    }
    return;
  }

  if (wid <= NSW) {
    // ===================== stream: block bounds U_b, the row's max logit ====
    const int grp = (wid - 1) / GW, w = (wid - 1) % GW;
    uint64_t kc = 0;
    int64_t u = 0;
    for (;; ++u) {
      // the row id: read after this group's first chunk of the row has landed
      // (the producer wrote it before issuing that chunk, and can be at most
      // NR - 1 rows ahead: it reuses a stage only after both groups consumed
      // a later chunk than their first one of row u)
      const uint64_t kf = kc + (uint64_t)((grp - (int)(kc % NG) + NG) % NG);
      mbar_wait(&ring_full[kf % NST], (uint32_t)((kf / NST) & 1));
      const int64_t row = row_of[u % NR];
      const int sb = (int)(u % NS);
      const uint32_t suse = (uint32_t)(u / NS);
      if (suse > 0) SRT_TIMED(tw1, mbar_wait(&sum_free[sb], (suse - 1) & 1));
      if (row < 0) {  // past the last row: pass the end on to the tail
        if (lane == 0 && atomicAdd(&p1cnt[sb], 1u) == NSW - 1) {
          rowid[sb] = -1;
          mbar_arrive(&sum_ready[sb]);
        }
        break;
      }
      float* U = reinterpret_cast<float*>(sums + sb * a.sum_bytes);
      const uint4 meta = meta_p[u % NR];
      const uint32_t pos = meta.x, s_lo = meta.y, s_hi = meta.z;
      float tmax = -INFINITY;
      uint32_t tblk = 0xFFFFFFFFu;
      bool nan = false;
      for (uint32_t ch = 0; ch < nch; ++ch, ++kc) {
        if (NG > 1 && (int)(kc % NG) != grp) continue;  // the other group's chunk
        const int s = (int)(kc % NST);
        if (a.spin) mbar_spin(&ring_full[s], (uint32_t)((kc / NST) & 1));
        else SRT_TIMED(tw0, mbar_wait(&ring_full[s], (uint32_t)((kc / NST) & 1)));
        const int32_t left = (int32_t)(row_bytes - (int64_t)ch * CHUNK);
        const int32_t nb = left < (int32_t)CHUNK ? left : (int32_t)CHUNK;
        const int32_t npairs = (a.debug & 32) ? 0 : (nb + PAIRB - 1) / PAIRB;  // (32: timing probe)
        const unsigned char* st = ring + s * CHUNK;
        // (the Philox call is issued next to the shared loads, so its ALU work
        // hides their latency; measured faster than drawing it before the wait
        // and releasing the stage before the bound arithmetic)
        for (int32_t pi = w * 32 + lane; pi < npairs; pi += GW * 32) {
          const uint32_t gp = ch * PAIRS_PER_CHUNK + (uint32_t)pi;  // pair index in the row
          const int nA = block_len32(a.V, 2 * (int32_t)gp);
          const int nB = block_len32(a.V, 2 * (int32_t)gp + 1);
          const unsigned char* pa = st + pi * PAIRB;
          float mA, mB;
          if (nA == NOISE_BLK && nB == NOISE_BLK) {
            mA = block_max_nan<DT>(pa, lane);
            mB = block_max_nan<DT>(pa + BLKB, lane);
            if (mA != mA) { nan = true; mA = block_max_scalar<DT>(pa, NOISE_BLK); }
            if (mB != mB) { nan = true; mB = block_max_scalar<DT>(pa + BLKB, NOISE_BLK); }
          } else {  // the row's last, partial pair
            mA = block_max_scalar<DT>(pa, nA);
            mB = nB ? block_max_scalar<DT>(pa + BLKB, nB) : -INFINITY;
            for (int j = 0; j < nA; ++j) nan |= load_x<DT>(pa, j) != load_x<DT>(pa, j);
            for (int j = 0; j < nB; ++j)
              nan |= load_x<DT>(pa + BLKB, j) != load_x<DT>(pa + BLKB, j);
          }
          const Philox4 pw = philox4x32_10(0x80000000u | gp, pos, s_lo, s_hi, k0, k1);
          const float xa = unit_t ? mA : __fdiv_rn(mA, T);
          float GA;
          if (nA == NOISE_BLK) GA = tab[pw.x >> 22];  // bucket bound of G_b (r >> 13)
          else GA = block_noise(pw.x, pw.y, (uint32_t)nA).G;
          U[2 * gp] = __fadd_rn(xa, GA);
          if (mA > tmax || (tblk == 0xFFFFFFFFu && mA == mA)) { tmax = mA; tblk = 2 * gp; }
          if (nB) {
            const float xb = unit_t ? mB : __fdiv_rn(mB, T);
            float GB;
            if (nB == NOISE_BLK) GB = tab[pw.z >> 22];
            else GB = block_noise(pw.z, pw.w, (uint32_t)nB).G;
            U[2 * gp + 1] = __fadd_rn(xb, GB);
            if (mB > tmax) { tmax = mB; tblk = 2 * gp + 1; }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring_empty[s]);
      }
      if (__any_sync(0xffffffffu, nan) && lane == 0) set_error(c, SRT_DEV_NONFINITE_LOGIT);
      // (max logit desc, block asc) -> the CTA's packed row header
      const uint32_t mykey = tblk == 0xFFFFFFFFu ? 0u : fkey(tmax);
      const uint32_t wkey = __reduce_max_sync(0xffffffffu, mykey);
      const uint32_t wblk =
          __reduce_min_sync(0xffffffffu, (wkey && mykey == wkey) ? tblk : 0xFFFFFFFFu);
      __syncwarp();
      if (lane == 0) {
        if (wkey) atomicMax(&p1key[sb], ((unsigned long long)wkey << 32) | (0xFFFFFFFFu - wblk));
        __threadfence_block();
        if (atomicAdd(&p1cnt[sb], 1u) == NSW - 1) {  // the last stream warp publishes
          rowhdr[sb] = atomicExch(&p1key[sb], 0ull);
          rowid[sb] = row;
          meta_s[sb] = meta;
          p1cnt[sb] = 0;
          mbar_arrive(&sum_ready[sb]);  // release: the summary is complete
        }
      }
    }
    SRT_PROF_PRINT("stream");
    return;
  }

  // ======================= tail: M, then the surviving blocks ==============
  // Tail warp 0 (the M warp) runs ahead of the others: for each row it finds
  // i* (the first element of the row's max-logit block equal to the row's
  // max logit) and publishes M = z(i*) in rowM, then releases the row to the
  // workers (m_ready).  Its global load and noise arithmetic are thus off the
  // workers' per-row chain.
  if (wid == 1 + NSW) {
    for (int64_t u = 0;; ++u) {
      const int sb = (int)(u % NS);
      SRT_TIMED(tw0, mbar_wait(&sum_ready[sb], (uint32_t)((u / NS) & 1)));
      const int64_t row = rowid[sb];
      if (row < 0) {  // the end: pass it on to the workers
        __syncwarp();
        if (lane == 0) mbar_arrive(&m_ready[sb]);
        break;
      }
      const unsigned long long hdr = rowhdr[sb];
      uint32_t mkey = 0u;  // (none: every logit of the row is NaN)
      if (hdr != 0 && !(a.debug & 16)) {
        const uint4 meta = meta_s[sb];
        const uint32_t pos = meta.x, s_lo = meta.y, s_hi = meta.z;
        const unsigned char* rowp = (const unsigned char*)a.logits + row * row_bytes;
        const float X = key_value((uint32_t)(hdr >> 32));
        const uint32_t bX = 0xFFFFFFFFu - (uint32_t)hdr;
        const int nX = block_len32(a.V, (int32_t)bX);
        const int64_t vX = (int64_t)bX * NOISE_BLK;
        uint32_t first = 0xFFFFFFFFu;
        if (2 * lane < nX && load_x<DT>(rowp, vX + 2 * lane) == X) first = 2 * lane;
        else if (2 * lane + 1 < nX && load_x<DT>(rowp, vX + 2 * lane + 1) == X) first = 2 * lane + 1;
        const uint32_t jstar = __reduce_min_sync(0xffffffffu, first);
        uint32_t wa, wb;
        block_words(bX, pos, s_lo, s_hi, k0, k1, wa, wb);
        const BlockNoise bn = block_noise(wa, wb, (uint32_t)nX);
        float g = bn.G;
        const int64_t vs = vX + jstar;
        if (jstar != bn.p) {
          const Philox4 pw = philox4x32_10((uint32_t)(vs >> 2), pos, s_lo, s_hi, k0, k1);
          const uint32_t k = (uint32_t)(vs & 3);
          g = element_noise_from_word(k == 0 ? pw.x : k == 1 ? pw.y : k == 2 ? pw.z : pw.w, bn);
        }
        mkey = fkey(perturbed(X, g, T, unit_t));  // M = z(i*) is never NaN
      }
      __syncwarp();
      if (lane == 0) {
        rowM[sb] = mkey;
        mbar_arrive(&m_ready[sb]);  // release: M and the row header
      }
    }
    SRT_PROF_PRINT("m-warp");
    return;
  }

  // Workers (NT - 1 warps): every block whose bound U_b reaches an achieved z.
  constexpr int NTW = NT - 1;
  const int t = wid - 2 - NSW;
  int64_t u = 0;
  for (;; ++u) {
    const int sb = (int)(u % NS);
    SRT_TIMED(tw0, mbar_wait(&m_ready[sb], (uint32_t)((u / NS) & 1)));
    const int64_t row = rowid[sb];
    if (row < 0) break;
    const unsigned long long hdr = rowhdr[sb];
    const float* U = reinterpret_cast<const float*>(sums + sb * a.sum_bytes);
    float bz = -INFINITY;
    int32_t bv = INT_MAX;
    if (hdr != 0 && !(a.debug & 16)) {  // else every logit NaN (debug 16: timing probe, no tail)
      const uint4 meta = meta_s[sb];
      const uint32_t pos = meta.x, s_lo = meta.y, s_hi = meta.z;
      const unsigned char* rowp = (const unsigned char*)a.logits + row * row_bytes;
      float M = key_value(*(volatile uint32_t*)&rowM[sb]);  // z(i*) from the M warp
      bool raised = false;  // M raised since this warp last shared it (share_M)
      // Exact evaluation of block b by the whole warp (lane = 2 consecutive
      // tokens, coalesced); the best (z, v) and M are raised as it goes.
      auto eval_block = [&](int32_t b, float2 xx) {
        const int n = block_len32(a.V, b);
        uint32_t wa, wb;
        block_words((uint32_t)b, pos, s_lo, s_hi, k0, k1, wa, wb);
        const BlockNoise bn = block_noise(wa, wb, (uint32_t)n);
        const float xs0 = unit_t ? xx.x : __fdiv_rn(xx.x, T);
        const float xs1 = unit_t ? xx.y : __fdiv_rn(xx.y, T);
        // g_v <= G_b: skip a token if even the block maximum cannot reach M
        const bool n0 = __fadd_rn(xs0, bn.G) >= M, n1 = __fadd_rn(xs1, bn.G) >= M;
        if (!(n0 || n1)) return;  // (NaN fails both tests)
        const int64_t v = (int64_t)b * NOISE_BLK + 2 * lane;
        const Philox4 pw = philox4x32_10((uint32_t)(v >> 2), pos, s_lo, s_hi, k0, k1);
        const bool hi = (lane & 1) != 0;  // tokens 2l, 2l+1 are words 0,1 or 2,3
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (!(k ? n1 : n0)) continue;
          const uint32_t j = 2 * lane + k;
          const uint32_t wd = hi ? (k ? pw.w : pw.z) : (k ? pw.y : pw.x);
          const float g = j == bn.p ? bn.G : element_noise_from_word(wd, bn);
          const float z = __fadd_rn(k ? xs1 : xs0, g);
          if (cand_better(z, (int32_t)(v + k), bz, bv)) {
            bz = z;
            bv = (int32_t)(v + k);
            if (z > M) { M = z; raised = true; }
          }
        }
      };
      auto load_block = [&](int32_t b) {
        const int n = block_len32(a.V, b);
        const int64_t v = (int64_t)b * NOISE_BLK + 2 * lane;
        float2 xx;
        xx.x = 2 * lane < n ? load_x<DT>(rowp, v) : NAN;
        xx.y = 2 * lane + 1 < n ? load_x<DT>(rowp, v + 1) : NAN;
        return xx;
      };
      // the warp's M joins the row's shared bound; the row's best M comes back.
      // Only a warp whose lanes raised M since they last shared it publishes
      // (warp max + one shared atomic); the others just read the pooled bound.
      auto share_M = [&]() {
        if (__any_sync(0xffffffffu, raised)) {
          const uint32_t wk = __reduce_max_sync(0xffffffffu, fkey(M));  // M is never NaN
          if (lane == 0) atomicMax(&rowM[sb], wk);
          __syncwarp();
          raised = false;
        }
        const uint32_t k = *(volatile uint32_t*)&rowM[sb];
        M = fmaxf(M, key_value(k));
      };
      const int32_t nchunk = (a.nblk + 31) / 32;
      // Phase 1 (branch and bound): each worker first evaluates the block of
      // its share with the largest bound U_b, which usually holds a z near
      // the row's maximum; the workers pool their M before phase 2, so far
      // fewer blocks pass U_b >= M than against z(i*) alone.
      int32_t b1 = -1;
      {
        uint32_t bu = 0;
        int32_t bi = INT_MAX;
        for (int32_t cb = t; cb < nchunk; cb += NTW) {
          const int32_t b = cb * 32 + lane;
          if (b < a.nblk) {
            const uint32_t k = fkey(U[b]);
            if (k > bu) { bu = k; bi = b; }
          }
        }
        const uint32_t wbu = __reduce_max_sync(0xffffffffu, bu);
        const int32_t wbi = __reduce_min_sync(0xffffffffu, (wbu && bu == wbu) ? bi : INT_MAX);
        if (wbu && U[wbi] >= M) {
          b1 = wbi;
          eval_block(b1, load_block(b1));
        }
      }
      share_M();
      SRT_TIMED(tw1, asm volatile("bar.sync 1, %0;" ::"r"(NTW * 32) : "memory"));
      share_M();
      // Phase 2: every other block whose bound reaches M, BATCH at a time so
      // their L2 loads overlap; M is re-pooled after each batch.
      constexpr int BATCH = 4;
      for (int32_t cb = t; cb < nchunk; cb += NTW) {
        const int32_t b = cb * 32 + lane;
        unsigned surv = __ballot_sync(0xffffffffu, b < a.nblk && b != b1 && U[b] >= M);
        while (surv) {
          int32_t bb[BATCH];
          float2 xx[BATCH];
#pragma unroll
          for (int i = 0; i < BATCH; ++i) {  // pop up to BATCH blocks, issue their loads
            bb[i] = -1;
            if (surv) {
              bb[i] = cb * 32 + __ffs(surv) - 1;
              surv &= surv - 1;
              xx[i] = load_block(bb[i]);
            }
          }
#pragma unroll
          for (int i = 0; i < BATCH; ++i)
            if (bb[i] >= 0 && U[bb[i]] >= M) eval_block(bb[i], xx[i]);
          if (surv) {
            share_M();
            surv &= __ballot_sync(0xffffffffu, b < a.nblk && U[b] >= M);
          }
        }
        share_M();
      }
    }
    const unsigned long long mine = bv == INT_MAX ? 0ull : pack_cand(bz, bv);
    const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(mine >> 32));
    const uint32_t lo32 =
        __reduce_max_sync(0xffffffffu, (uint32_t)(mine >> 32) == hi ? (uint32_t)mine : 0u);
    const unsigned long long wbest = ((unsigned long long)hi << 32) | lo32;
    __syncwarp();
    if (lane == 0) {
      if (wbest) atomicMax(&a.result[row], wbest);
      if (a.seq_done) {  // the row's last worker: its result is final
        __threadfence();
        if (atomicAdd(&wdone[sb], 1u) == NTW - 1) {
          wdone[sb] = 0;  // (before the arrival that frees the slot)
          __threadfence();
          atomicAdd(&a.seq_done[meta_s[sb].w], 1u);
        }
      }
      mbar_arrive(&sum_free[sb]);
    }
  }
  SRT_PROF_PRINT("tail");
  if (SRT_SCAN_PROF_ON && (a.debug & 128) && t == 0 && lane == 0) {  // per-CTA span (ns)
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    printf("[scan cta] %d %llu %llu %lld\n", blockIdx.x, g_start, g_end, u);
  }
#undef SRT_TIMED
#undef SRT_PROF_PRINT
}

// per row: (sequence, position) — rows of sequence s are [row_offsets[s],
// row_offsets[s+1]); also clears the row's packed result.  One warp per
// sequence, a lane per row.
__global__ void k_rowinfo(VerifyArgs a, int32_t Bmax, int2* rowinfo,
                          unsigned long long* result) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= a.n) return;
  const int64_t r0 = a.row_offsets[s];
  const int32_t t = a.seq_len[s];
  const int32_t nd = (int32_t)(a.row_offsets[s + 1] - r0 - 1);
  for (int32_t i = lane - 1; i < nd; i += 32) {
    rowinfo[r0 + 1 + i] = make_int2(s, i < 0 ? t : t + a.draft_depth[(int64_t)s * Bmax + i]);
    result[r0 + 1 + i] = 0;
  }
}

template <int DT, int NSW, int NT, int NST, int NS, uint32_t CHUNK, int NG>
cudaError_t launch_rows(const DevCache& c, ScanParams p, cudaStream_t stream) {
  constexpr int THREADS = (1 + NSW + NT) * 32;
  const size_t smem = (size_t)NST * CHUNK + (size_t)NS * p.sum_bytes +
                      (2 * NST + 3 * NS) * 8 + 2 * NS * 8 + (NS + NST + 2) * 8 +
                      2 * ((NS + 3) & ~3) * 4 +
                      NOISE_BUCKETS * 4 + ((NS + 3) & ~3) * 4 + (size_t)(NST + 2 + NS) * 16;
  auto kern = k_scan_rows<DT, NSW, NT, NST, NS, CHUNK, NG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  static int blocks = 0;
  if (!blocks) {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
    if (e != cudaSuccess || per_sm <= 0) per_sm = 1;
    blocks = per_sm * num_sms();
    if (const char* g = getenv("SRT_SCAN_GRID")) {  // development knob: fewer CTAs
      const int x = atoi(g);
      if (x > 0 && x < blocks) blocks = x;
    }
    if (p.debug & 8)
      fprintf(stderr, "[srt scan] rows: NSW=%d NT=%d NST=%d NS=%d CHUNK=%u NG=%d hint=%u spin=%u smem=%zu -> %d CTAs\n",
              NSW, NT, NST, NS, CHUNK, NG, p.l2_hint, p.spin, smem, blocks);
  }
  const int grid = p.grid_cap > 0 && p.grid_cap < blocks ? p.grid_cap : blocks;
  k_scan_rows<DT, NSW, NT, NST, NS, CHUNK, NG><<<grid, THREADS, smem, stream>>>(c, p);
  return cudaGetLastError();
}

}  // namespace

// The rows kernel serves every V whose rows are 16-byte multiples (TMA) and
// whose block summaries fit in shared memory; the rest takes the reference.
int scan_cluster_size(int32_t V, int dtype) {
  if ((int64_t)V * (dtype == SRT_BF16 ? 2 : 4) % 16) return 0;
  const int64_t nblk = ((int64_t)V + NOISE_BLK - 1) / NOISE_BLK;
  return nblk * 4 <= 16 * 1024 ? 1 : 0;
}

cudaError_t launch_rowinfo(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                           unsigned long long* result, cudaStream_t stream) {
  k_rowinfo<<<(a.n * 32 + 255) / 256, 256, 0, stream>>>(a, c.Bmax, rowinfo, result);
  return cudaGetLastError();
}

cudaError_t launch_scan_cluster(const DevCache& c, const VerifyArgs& a, int2* rowinfo,
                                unsigned long long* result, cudaStream_t stream) {
  if (!scan_cluster_size(c.V, a.dtype)) return cudaErrorInvalidValue;
  k_rowinfo<<<(a.n * 32 + 255) / 256, 256, 0, stream>>>(a, c.Bmax, rowinfo, result);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_scan_list(c, a, rowinfo, nullptr, a.row_offsets + a.n, result, stream);
}

// The rows kernel over rows row_list[0 .. *count) (or [0, *count) when
// row_list is null), rowinfo and result indexed by row id; result[row] must
// be 0 for every listed row.
cudaError_t launch_scan_list(const DevCache& c, const VerifyArgs& a, const int2* rowinfo,
                             const int32_t* row_list, const int64_t* count,
                             unsigned long long* result, cudaStream_t stream,
                             uint32_t* seq_done, int grid_cap) {
  if (!scan_cluster_size(c.V, a.dtype)) return cudaErrorInvalidValue;
  ScanParams p;
  p.seq_done = seq_done;
  p.grid_cap = grid_cap;
  p.logits = a.logits;
  p.rowinfo = rowinfo;
  p.row_list = row_list;
  p.total = count;
  p.seq_id = a.seq_id;
  p.seed = a.seed;
  p.temperature = a.temperature;
  p.result = result;
  p.V = c.V;
  p.nblk = (c.V + NOISE_BLK - 1) / NOISE_BLK;
  p.sum_bytes = (uint32_t)(((int64_t)p.nblk * 4 + 127) / 128 * 128);
  static int dbg = -1;
  if (dbg < 0) {
    const char* s = getenv("SRT_SCAN_DEBUG");
    dbg = s ? atoi(s) : 0;
  }
  p.debug = (uint32_t)dbg;
  // SRT_SCAN_ROWS="NSW,NT,NST,NS,CHUNK_KB,HINT,NG,SPIN" picks another
  // instantiated pipeline shape (development knob; tools/scan_sweep.sh)
  static int cfg[8] = {-1, 0, 0, 0, 0, 0, 0, 0};
  if (cfg[0] < 0) {
    // (HINT 0: no L2 policy on the streamed rows -- evict_first was +2-4 % in
    // the r01 probe but -2 to -4 % in every r02 step configuration)
    int d[8] = {8, 10, 4, 4, 32, 0, 2, 0};
    if (const char* s = getenv("SRT_SCAN_ROWS")) {
      int x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const int k = sscanf(s, "%d,%d,%d,%d,%d,%d,%d,%d", &x[0], &x[1], &x[2], &x[3], &x[4], &x[5],
                           &x[6], &x[7]);
      for (int i = 0; i < k; ++i) d[i] = x[i];
    }
    for (int i = 0; i < 8; ++i) cfg[i] = d[i];
  }
  p.l2_hint = (uint32_t)cfg[5];
  p.spin = (uint32_t)cfg[7];
  // rows claimed dynamically (SRT_SCAN_STATIC=1: the static interleave)
  static int stat = -1;
  if (stat < 0) {
    const char* e = getenv("SRT_SCAN_STATIC");
    stat = e ? atoi(e) : 0;
  }
  p.sched = stat ? nullptr : c.sched;
#define SRT_ROWS_CASE(A, B, C, D, K, G)                                                            \
  if (cfg[0] == A && cfg[1] == B && cfg[2] == C && cfg[3] == D && cfg[4] == K && cfg[6] == G)     \
    return a.dtype == SRT_BF16 ? launch_rows<SRT_BF16, A, B, C, D, K * 1024u, G>(c, p, stream)    \
                               : launch_rows<SRT_F32, A, B, C, D, K * 1024u, G>(c, p, stream);
  SRT_ROWS_CASE(4, 12, 4, 4, 32, 1)
  SRT_ROWS_CASE(8, 8, 4, 4, 32, 2)
  SRT_ROWS_CASE(8, 12, 4, 4, 32, 2)
  SRT_ROWS_CASE(8, 11, 4, 4, 32, 2)
  SRT_ROWS_CASE(8, 10, 6, 2, 32, 2)
  SRT_ROWS_CASE(8, 10, 6, 3, 32, 2)
  SRT_ROWS_CASE(12, 8, 6, 2, 32, 3)
  SRT_ROWS_CASE(12, 9, 6, 3, 32, 3)
#undef SRT_ROWS_CASE
  return a.dtype == SRT_BF16 ? launch_rows<SRT_BF16, 8, 10, 4, 4, 32768u, 2>(c, p, stream)
                             : launch_rows<SRT_F32, 8, 10, 4, 4, 32768u, 2>(c, p, stream);
}

}  // namespace srt
