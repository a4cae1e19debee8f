// cache.cu — cache initialisation, the exact noise-bound tables, the noise
// table test hook and the dump enumeration kernel.
#include "noise.cuh"
#include "srt_internal.cuh"

namespace srt {

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

__global__ void k_init_counters(DevCache c) {
  c.ctr[0] = (unsigned long long)c.P;  // the roots (node ids H .. H+P-1)
  c.ctr[1] = 0;
  *c.status = 0;
}

cudaError_t launch_init_cache(const DevCache& c, cudaStream_t stream) {
  cudaError_t e;
  const size_t NN = c.H + (size_t)c.P;  // node ids: hash slots, then the roots
  if ((e = cudaMemsetAsync(c.tok, 0xFF, NN * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.cnt, 0, NN * 4, stream)) != cudaSuccess) return e;
  // rec = {nchild 0, child0 -, token -, csum 0 | no blocks}: child0 is read only
  // if nchild >= 1
  if ((e = cudaMemsetAsync(c.rec, 0, NN * 32, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.hash, 0xFF, c.H * sizeof(HashSlot), stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.slots, 0xFF, c.W * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.stok, 0xFF, c.W * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.scnt, 0, c.W * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.hub_node, 0xFF, (size_t)c.HC * 4, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.hub_claim, 0, (size_t)c.HC * 8, stream)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c.dirty_n, 0, 8, stream)) != cudaSuccess) return e;
  k_init_counters<<<1, 1, 0, stream>>>(c);
  return cudaGetLastError();
}

// The maximum noise of a FULL 64-token block as a function of its word's
// r = wa >> 9:  G64(r) = -log_det(RN(-log_det(u(r)) / 64))  (O11).
// Bucket b covers r in [b << 13, (b+1) << 13): gbound[b] = max G64 over the
// bucket, gbound[1024] = max over all r, gbound[2049 + b] = max over the
// bucket of the single-word Gumbel g(r) = -log_det(-log_det(u(r))) (the
// fused LM-head sampler's per-element pre-bound), gbound[1025 + b] = min over the
// bucket.  Computed by enumeration, so the bounds are exact whatever the shape
// of G64; the scan's block bound is max x + gbound[r >> 13].
__global__ void __launch_bounds__(256) k_noise_bucket_max(float* gbound) {
  __shared__ float red[8], redmin[8];
  const uint32_t b = blockIdx.x;
  __shared__ float redg[8];
  float m = -INFINITY, mn = INFINITY, mg = -INFINITY;
  for (uint32_t j = threadIdx.x; j < (1u << NOISE_BUCKET_SHIFT); j += blockDim.x) {
    const uint32_t r = (b << NOISE_BUCKET_SHIFT) | j;
    const BlockNoise bn = block_noise(r << 9, 0u, (uint32_t)NOISE_BLK);
    const float g = bn.G;
    m = fmaxf(m, g);
    mn = fminf(mn, g);
    mg = fmaxf(mg, gumbel_of_r(r));
  }
  for (int o = 16; o; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = m;
    redmin[threadIdx.x >> 5] = mn;
    redg[threadIdx.x >> 5] = mg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      m = fmaxf(m, red[w]);
      mn = fminf(mn, redmin[w]);
      mg = fmaxf(mg, redg[w]);
    }
    gbound[b] = m;
    gbound[NOISE_BUCKETS + 1 + b] = mn;
    gbound[2 * NOISE_BUCKETS + 1 + b] = mg;
  }
}

__global__ void k_noise_global_max(float* gbound) {
  float m = -INFINITY;
  for (int b = threadIdx.x; b < NOISE_BUCKETS; b += 32) m = fmaxf(m, gbound[b]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) gbound[NOISE_BUCKETS] = m;
}

cudaError_t launch_noise_bounds(const DevCache& c, cudaStream_t stream) {
  k_noise_bucket_max<<<NOISE_BUCKETS, 256, 0, stream>>>(c.gbound);
  k_noise_global_max<<<1, 32, 0, stream>>>(c.gbound);
  return cudaGetLastError();
}

__global__ void k_noise_table(float* out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < (1u << 23)) out[r] = gumbel_of_r(r);
}

cudaError_t launch_noise_table(float* out, cudaStream_t stream) {
  k_noise_table<<<(1u << 23) / 256, 256, 0, stream>>>(out);
  return cudaGetLastError();
}

// log_det of the floats with bit patterns first, first + 1, ... (test hook:
// the exhaustive device/oracle comparison of O12 over the positive normals).
__global__ void k_log_det_range(uint32_t first, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = log_det(__uint_as_float(first + (uint32_t)i));
}

cudaError_t launch_log_det_range(uint32_t first, int64_t n, float* out, cudaStream_t stream) {
  k_log_det_range<<<num_sms() * 8, 256, 0, stream>>>(first, n, out);
  return cudaGetLastError();
}

// g_v of every element of the rows keyed (seq_id[k], pos[k]): the O11 block
// construction through the same device functions the scan evaluates (one
// block of 64 tokens per warp-pair of lanes; test hook).
__global__ void k_row_noise(int32_t V, uint64_t seed, const uint64_t* seq_id, const int32_t* pos,
                            int32_t nkeys, float* out) {
  const int64_t nblk = ((int64_t)V + NOISE_BLK - 1) / NOISE_BLK;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nkeys * nblk;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = (int32_t)(t / nblk);
    const int64_t b = t % nblk;
    const uint64_t sid = seq_id[key];
    const uint32_t ps = (uint32_t)pos[key], slo = (uint32_t)sid, shi = (uint32_t)(sid >> 32);
    const int n = block_len(V, b);
    uint32_t wa, wb;
    block_words((uint32_t)b, ps, slo, shi, k0, k1, wa, wb);
    const BlockNoise bn = block_noise(wa, wb, (uint32_t)n);
    float* g = out + (int64_t)key * V + b * NOISE_BLK;
    for (int j = 0; j < n; ++j) {
      if ((uint32_t)j == bn.p) {
        g[j] = bn.G;
        continue;
      }
      const int64_t v = b * NOISE_BLK + j;
      const Philox4 pw = philox4x32_10((uint32_t)(v >> 2), ps, slo, shi, k0, k1);
      const uint32_t q = (uint32_t)(v & 3);
      g[j] = element_noise_from_word(q == 0 ? pw.x : q == 1 ? pw.y : q == 2 ? pw.z : pw.w, bn);
    }
  }
}

cudaError_t launch_row_noise(int32_t V, uint64_t seed, const uint64_t* seq_id, const int32_t* pos,
                             int32_t nkeys, float* out, cudaStream_t stream) {
  k_row_noise<<<num_sms() * 8, 128, 0, stream>>>(V, seed, seq_id, pos, nkeys, out);
  return cudaGetLastError();
}

// One thread per frontier node: emit every child (test path only).  Children
// k >= 1 are read through their slot mirrors (stok, scnt: what srt_draft
// enumerates) and checked against the node arrays (tok, cnt).
__global__ void k_dump_level(DevCache c, const uint32_t* frontier, int32_t nf, uint32_t* out_node,
                             int32_t* out_parent, int32_t* out_tok, uint32_t* out_cnt,
                             uint32_t* out_nchild, unsigned int* out_n) {
  const int32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const uint32_t u = frontier[f];
  const uint4 r = *rec_of(c, u);
  const uint32_t F = r.x;
  for (uint32_t k = 0; k < F; ++k) {
    uint32_t ch;
    int32_t tk;
    uint32_t n;
    if (k == 0) {
      ch = r.y;
      tk = (int32_t)r.z;
      n = c.cnt[ch];
    } else {
      const uint32_t j = k - 1, i = blk_index(j);
      const uint32_t pos = block_base(c, u, i) + (j - blk_start(i));
      ch = c.slots[pos];
      tk = c.stok[pos];
      n = c.scnt[pos];
    }
    if (tk != c.tok[ch] || n != c.cnt[ch]) set_error(c, SRT_DEV_INCONSISTENT);
    const unsigned int o = atomicAdd(out_n, 1u);
    out_node[o] = ch;
    out_parent[o] = f;
    out_tok[o] = tk;
    out_cnt[o] = n;
    out_nchild[o] = rec_of(c, ch)->x;
  }
}

cudaError_t launch_dump_level(const DevCache& c, const uint32_t* frontier, int32_t nf,
                              uint32_t* out_node, int32_t* out_parent, int32_t* out_tok,
                              uint32_t* out_cnt, uint32_t* out_nchild, unsigned int* out_n,
                              cudaStream_t stream) {
  k_dump_level<<<(nf + 127) / 128, 128, 0, stream>>>(c, frontier, nf, out_node, out_parent,
                                                      out_tok, out_cnt, out_nchild, out_n);
  return cudaGetLastError();
}

}  // namespace srt
