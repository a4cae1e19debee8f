// stream_probe.cu — development micro-benchmark (not part of libsrt): how fast
// can a persistent kernel stream a multi-GB buffer through shared memory on
// this B200?  TMA 1-D bulk copies with NBUF stages of CHUNK bytes per CTA and
// K CTAs per SM, versus plain 16-byte LDG streaming.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void k_tma(const char* src, size_t total, uint32_t chunk, int nbuf,
                      unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nbuf * chunk);
  const size_t nchunks = total / chunk;
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbuf; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int b, size_t ci) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])),
                 "r"(chunk) : "memory");
    for (uint32_t off = 0; off < chunk; off += 32768) {
      uint32_t nb = chunk - off < 32768 ? chunk - off : 32768;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
          "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sm + (size_t)b * chunk + off)),
          "l"(src + ci * chunk + off), "r"(nb), "r"(smem_u32(&bar[b])), "l"(pol)
          : "memory");
    }
  };
  size_t first = blockIdx.x;
  if (threadIdx.x == 0)
    for (int b = 0; b < nbuf; ++b)
      if (first + (size_t)b * gridDim.x < nchunks) issue(b, first + (size_t)b * gridDim.x);
  unsigned long long acc = 0;
  size_t u = 0;
  for (size_t ci = first; ci < nchunks; ci += gridDim.x, ++u) {
    int b = (int)(u % nbuf);
    uint32_t ph = (uint32_t)((u / nbuf) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar[b])),
        "r"(ph)
        : "memory");
    // touch one 16 B vector per thread (keeps the data "used")
    const uint4 v = reinterpret_cast<const uint4*>(sm + (size_t)b * chunk)[threadIdx.x];
    acc += v.x ^ v.w;
    __syncthreads();
    if (threadIdx.x == 0) {
      size_t nx = ci + (size_t)nbuf * gridDim.x;
      if (nx < nchunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(b, nx);
      }
    }
  }
  if (acc == 0x123456789ull) *sink = acc;
}

__global__ void k_ldg(const uint4* src, size_t n, unsigned long long* sink) {
  unsigned long long acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; i < n; i += stride) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    acc += v.x ^ v.w;
  }
  if (acc == 0x123456789ull) *sink = acc;
}

int main() {
  const size_t total = 8ull << 30;  // 8 GiB
  char* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 3.0 * total / (ms / 1000.0) / 1e9;
  };
  for (int thr : {256, 512}) {
    for (int blocks_per_sm : {1, 2, 4, 8}) {
      double gbs = time_it([&] {
        k_ldg<<<sms * blocks_per_sm, thr>>>((const uint4*)buf, total / 16, sink);
      });
      printf("LDG  thr %d  blocks/SM %d : %7.1f GB/s\n", thr, blocks_per_sm, gbs);
    }
  }
  for (uint32_t chunk : {8192u, 16384u, 32768u, 65536u}) {
    for (int nbuf : {2, 3, 4, 6, 8}) {
      size_t smem = (size_t)nbuf * chunk + 8 * nbuf;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int k : {1, 2, 4}) {
        if (smem * k > 228 * 1024) continue;
        double gbs = time_it([&] { k_tma<<<sms * k, 256, smem>>>(buf, total, chunk, nbuf, sink); });
        cudaError_t err = cudaGetLastError();
        printf("TMA  chunk %6u nbuf %d ctas/SM %d (in flight/SM %4zu KB): %7.1f GB/s %s\n", chunk,
               nbuf, k, smem * k / 1024, gbs, err ? cudaGetErrorString(err) : "");
      }
    }
  }
  return 0;
}
