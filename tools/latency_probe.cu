// latency_probe.cu — development micro-benchmark (not part of libsrt): the
// round-trip latency of dependent random 16-byte loads (pointer chasing) as a
// function of the footprint, to see where TLB reach ends on this B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe latency_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_init(uint64_t* buf, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    buf[i] = (z ^ (z >> 31)) % n;  // next index: a random walk
  }
}

__global__ void k_chase(const uint64_t* buf, int steps, uint64_t start, long long* out, uint64_t* sink) {
  uint64_t i = (start + threadIdx.x * 7919ull + blockIdx.x * 104729ull) % 1000003ull;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(buf + i));
    i = v;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / steps;
  if (i == 0xFFFFFFFFFFFFull) *sink = i;
}

// dependent chain of atomic CAS (never succeeding: compare value absent) and
// of relaxed.gpu 32-byte loads, for comparison with plain loads
__global__ void k_chase_cas(uint64_t* buf, int steps, uint64_t start, long long* out, uint64_t* sink, int mode) {
  uint64_t i = (start + threadIdx.x * 7919ull + blockIdx.x * 104729ull) % 1000003ull;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    uint64_t v;
    if (mode == 0) {
      v = atomicCAS((unsigned long long*)(buf + i), 0xFFFFFFFFFFFFFFFFull, 0ull);
    } else {
      uint64_t a, b, c, d;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(buf + (i & ~3ull)));
      v = (i & 3) == 0 ? a : (i & 3) == 1 ? b : (i & 3) == 2 ? c : d;
    }
    i = v;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / steps;
  if (i == 0xFFFFFFFFFFFFull) *sink = i;
}

int main() {
  long long* out;
  uint64_t* sink;
  cudaMalloc(&out, 1024 * sizeof(long long));
  cudaMalloc(&sink, 8);
  for (size_t mb : {16, 128, 512, 2048, 8192, 32768}) {
    size_t n = mb * (1ull << 20) / 8;
    uint64_t* buf;
    if (cudaMalloc(&buf, n * 8) != cudaSuccess) { printf("alloc %zu MB failed\n", mb); break; }
    k_init<<<1184, 256>>>(buf, n, mb);
    for (int mode : {0, 1}) {
      for (int warps : {1, 148}) {
        k_chase_cas<<<warps, 32>>>(buf, 64, 1, out, sink, mode);
        k_chase_cas<<<warps, 32>>>(buf, 256, 2, out, sink, mode);
        long long h[1024];
        cudaMemcpy(h, out, warps * sizeof(long long), cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < warps; ++i) m += h[i];
        printf("footprint %6zu MB, %4d warps: %s %6.0f cycles per dependent op\n", mb, warps,
               mode == 0 ? "CAS           " : "ld.v4.u64 gpu ", m / warps);
      }
    }
    for (int warps : {1, 148}) {
      k_chase<<<warps, 32>>>(buf, 64, 1, out, sink);  // warm
      k_chase<<<warps, 32>>>(buf, 256, 2, out, sink);
      long long h[1024];
      cudaMemcpy(h, out, warps * sizeof(long long), cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < warps; ++i) m += h[i];
      printf("footprint %6zu MB, %4d warps x 32 lanes: %6.0f cycles per dependent load\n", mb, warps, m / warps);
    }
    cudaFree(buf);
  }
  return 0;
}
