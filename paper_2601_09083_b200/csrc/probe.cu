// probe.cu — measurement support (not on the SRT path): a read-only stream of
// a device buffer through shared memory with 1-D TMA bulk copies, the
// denominator bench.py reports the scan's bandwidth against alongside the
// copy peak ("a read-only streaming kernel measured in the same
// run").  Persistent, one CTA per SM (x ctas_per_sm), nbuf stages of `chunk`
// bytes each; the data is only touched (one 16-byte vector per thread per
// stage) so the kernel is bound by HBM reads alone.
#include <cstdint>

#include "srt_internal.cuh"

namespace srt {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(256) k_stream_read(const char* src, int64_t total,
                                                     uint32_t chunk, int nbuf,
                                                     unsigned long long* sink, int hint) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nbuf * chunk);
  const int64_t nchunks = total / chunk;
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbuf; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // L2 policy of the copies: none (the scan's default since r02 v5, measured
  // faster in the step) or evict_first (SRT_STREAM_HINT=1)
  uint64_t pol = 0;
  if (hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int b, int64_t ci) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[b])),
                 "r"(chunk)
                 : "memory");
    for (uint32_t off = 0; off < chunk; off += 32768) {
      const uint32_t nb = chunk - off < 32768 ? chunk - off : 32768;
      if (hint)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(sm + (size_t)b * chunk + off)),
            "l"(src + ci * chunk + off), "r"(nb), "r"(smem_addr(&bar[b])), "l"(pol)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1], %2, [%3];" ::"r"(smem_addr(sm + (size_t)b * chunk + off)),
            "l"(src + ci * chunk + off), "r"(nb), "r"(smem_addr(&bar[b]))
            : "memory");
    }
  };
  const int64_t first = blockIdx.x;
  if (threadIdx.x == 0)
    for (int b = 0; b < nbuf; ++b)
      if (first + (int64_t)b * gridDim.x < nchunks) issue(b, first + (int64_t)b * gridDim.x);
  unsigned long long acc = 0;
  int64_t u = 0;
  for (int64_t ci = first; ci < nchunks; ci += gridDim.x, ++u) {
    const int b = (int)(u % nbuf);
    const uint32_t ph = (uint32_t)((u / nbuf) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_addr(&bar[b])),
        "r"(ph)
        : "memory");
    const uint4 v = reinterpret_cast<const uint4*>(sm + (size_t)b * chunk)[threadIdx.x];
    acc += v.x ^ v.w;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t nx = ci + (int64_t)nbuf * gridDim.x;
      if (nx < nchunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(b, nx);
      }
    }
  }
  if (acc == 0x123456789ull) *sink = acc;
}

}  // namespace

cudaError_t launch_stream_read(const void* buf, int64_t bytes, int32_t chunk, int32_t nbuf,
                               int32_t ctas_per_sm, unsigned long long* sink,
                               cudaStream_t stream) {
  const size_t smem = (size_t)nbuf * chunk + 8 * (size_t)nbuf;
  cudaError_t e = cudaFuncSetAttribute(k_stream_read, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  static int hint = -1;
  if (hint < 0) {
    const char* h = getenv("SRT_STREAM_HINT");
    hint = h ? atoi(h) : 0;
  }
  k_stream_read<<<num_sms() * ctas_per_sm, 256, smem, stream>>>((const char*)buf, bytes,
                                                                 (uint32_t)chunk, nbuf, sink, hint);
  return cudaGetLastError();
}

}  // namespace srt
