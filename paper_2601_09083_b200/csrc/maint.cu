// maint.cu — capacity management of the trees (O17):
// prune by count threshold (the lowest-count subtrees go first: count(u) >=
// the count of each child, O1, so {count < theta} is closed under
// descendants), the count histogram that picks theta for eviction with
// hysteresis, and the level kernels of the dump load (persistence).
//
// Prune is a level-synchronous BFS driven by the host (srt_cache_prune):
//   k_prune_level: one warp per kept node; its children are classified and the
//     kept ones compacted in place (inline child 0, then the child-block
//     slots; moved children get their new slot word in their hash aux, their
//     count mirror and token; nchild and csum are rewritten), kept children go
//     to the next kept frontier, the others to the dead frontier;
//   k_kill_level: one thread per dead node: its children join the dead
//     frontier, its edge slot and child-block keys >= 4 become tombstones
//     (never matched, never EMPTY, so every probe sequence stays intact), its
//     record is cleared.
// Maintenance, not the per-step path: blocking, latency irrelevant.
#include "srt_internal.cuh"

namespace srt {

namespace {

// Slot word of child k >= 1 of u (blocks via the record or the hash).
__device__ __forceinline__ uint32_t child_pos(const DevCache& c, uint32_t u, uint32_t k) {
  const uint32_t j = k - 1, i = blk_index(j);
  return block_base(c, u, i) + (j - blk_start(i));
}

__global__ void k_prune_level(DevCache c, const uint32_t* __restrict__ front, int32_t nf,
                              uint32_t theta, uint32_t* __restrict__ next_keep, unsigned* n_keep,
                              uint32_t* __restrict__ next_dead, unsigned* n_dead) {
  const int lane = threadIdx.x & 31;
  const int32_t f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (f >= nf) return;
  const uint32_t u = front[f];
  uint4* rp = rec_of(c, u);
  const uint4 r = *rp;
  const uint32_t nch = r.x;
  uint32_t kept = 0;
  unsigned long long csum = 0;
  for (uint32_t kb = 0; kb < nch; kb += 32) {
    const uint32_t k = kb + lane;
    const bool valid = k < nch;
    uint32_t id = NONE, cn = 0;
    int32_t tk = -1;
    if (valid) {
      if (k == 0) {
        id = r.y;
        tk = (int32_t)r.z;
      } else {
        const uint32_t pos = child_pos(c, u, k);
        id = c.slots[pos];
        tk = c.stok[pos];
      }
      cn = c.cnt[id];
    }
    const bool keep = valid && cn >= theta;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    const uint32_t newk = kept + __popc(km & lanemask_lt());
    __syncwarp();  // every read of this chunk before any write (newk <= k)
    if (keep) {
      if (newk == 0) {
        rp->y = id;
        rp->z = (uint32_t)tk;
        c.hash[id].aux = AUX_CHILD0;
      } else {
        const uint32_t p2 = child_pos(c, u, newk);
        c.slots[p2] = id;
        c.stok[p2] = tk;
        c.scnt[p2] = cn;
        c.hash[id].aux = p2;
      }
      next_keep[atomicAdd(n_keep, 1u)] = id;
    } else if (valid) {
      next_dead[atomicAdd(n_dead, 1u)] = id;
    }
    unsigned long long s = keep ? cn : 0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    csum += s;
    kept += __popc(km);
    __syncwarp();
  }
  // vacated slots start clean for the children attached later (their count
  // mirrors are incremented from here)
  for (uint32_t k = max(kept, 1u) + lane; k < nch; k += 32) {
    const uint32_t pos = child_pos(c, u, k);
    c.slots[pos] = NONE;
    c.stok[pos] = -1;
    c.scnt[pos] = 0;
  }
  if (lane == 0 && kept != nch) {
    rp->x = kept;
    rp->w = (uint32_t)csum;
  }
}

__global__ void k_kill_level(DevCache c, const uint32_t* __restrict__ dead, int32_t nd,
                             uint32_t* __restrict__ next_dead, unsigned* n_dead,
                             unsigned long long* removed) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nd) return;
  const uint32_t v = dead[i];
  uint4* rp = rec_of(c, v);
  const uint4 r = *rp;
  const uint32_t nch = r.x;
  for (uint32_t k = 0; k < nch; ++k)
    next_dead[atomicAdd(n_dead, 1u)] = k == 0 ? r.y : c.slots[child_pos(c, v, k)];
  if (nch >= 2)
    for (uint32_t b = 4; b <= blk_index(nch - 2); ++b) {
      const uint32_t h = hash_slot(c, block_key(v, b));
      if (h != NONE) c.hash[h].key = TOMB_KEY;
    }
  c.hash[v].key = TOMB_KEY;  // the node's own edge (its id is the slot)
  c.tok[v] = -1;
  c.cnt[v] = 0;
  rp[0] = make_uint4(0, 0, 0, 0);
  rp[1] = make_uint4(0, 0, 0, 0);
  atomicAdd(removed, 1ull);
}

// hist[min(count, nb - 1)] over every live node (edge slots of the hash).
__global__ void k_count_hist(DevCache c, unsigned long long* hist, int32_t nb) {
  for (unsigned long long h = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; h < c.H;
       h += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k = c.hash[h].key;
    if (k == EMPTY_KEY || k == TOMB_KEY || ((uint32_t)k & BLOCK_TAG)) continue;
    const uint32_t n = c.cnt[h];
    atomicAdd(&hist[n < (uint32_t)nb ? n : (uint32_t)(nb - 1)], 1ull);
  }
}

}  // namespace

cudaError_t launch_prune_level(const DevCache& c, const uint32_t* front, int32_t nf, uint32_t theta,
                               uint32_t* next_keep, unsigned* n_keep, uint32_t* next_dead,
                               unsigned* n_dead, cudaStream_t stream) {
  if (nf <= 0) return cudaSuccess;
  const int64_t threads = (int64_t)nf * 32;
  k_prune_level<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(c, front, nf, theta, next_keep,
                                                                         n_keep, next_dead, n_dead);
  return cudaGetLastError();
}

cudaError_t launch_kill_level(const DevCache& c, const uint32_t* dead, int32_t nd,
                              uint32_t* next_dead, unsigned* n_dead, unsigned long long* removed,
                              cudaStream_t stream) {
  if (nd <= 0) return cudaSuccess;
  k_kill_level<<<(nd + 255) / 256, 256, 0, stream>>>(c, dead, nd, next_dead, n_dead, removed);
  return cudaGetLastError();
}

cudaError_t launch_count_hist(const DevCache& c, unsigned long long* hist, int32_t nb,
                              cudaStream_t stream) {
  k_count_hist<<<num_sms() * 8, 256, 0, stream>>>(c, hist, nb);
  return cudaGetLastError();
}

}  // namespace srt
