// k_shard.cu -- stage-1 exchange of the key-hash-sharded map.
//
// Stage 1 (A1-A5) is frame-parallel: shard g runs it for the window slots i = g + G j.  Its
// results then go where stage 2 needs them:
//  * the per-detection records (status, |V_s|, Q factors, e_s, t_s, key AABB, area, bbox) and the
//    frame's meta (S, frame id, key_out_of_range) to EVERY shard (all-gather: the association is
//    replicated on identical inputs);
//  * each unique (s, key) pair of a kept detection to the shard that OWNS the key
//    (owner = key_owner(key, G), all-to-all): lookups, inserts and relabels touch own keys only.
#include "disc_common.cuh"
#include "disc_launch.h"

namespace disc {

struct MetaArr { FrameMeta m[MAXWIN]; };

__global__ void k_det_pack(WinBufs src, int n, MetaArr meta, uint8_t* buf, DetLayout L, int Df, int Dt, int sem) {
  const int j = blockIdx.y;
  if (j >= n) return;
  uint8_t* rec = buf + (size_t)j * L.total;
  const int S = meta.m[j].S;
  const size_t fo = (size_t)j * src.SMAX;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t* mt = (int64_t*)(rec + L.meta);
    mt[0] = S;
    mt[1] = meta.m[j].frame_id;
    mt[2] = (int64_t)src.oor[j];
  }
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int s = tid; s < S; s += nt) {
    ((int32_t*)(rec + L.status))[s] = src.status[fo + s];
    ((uint32_t*)(rec + L.vs))[s] = src.vs[fo + s];
    ((uint32_t*)(rec + L.area))[s] = src.area[fo + s];
    rec[L.tok + s] = src.tok[fo + s];
    for (int k = 0; k < 6; ++k) {
      ((float*)(rec + L.qf))[6 * s + k] = src.qf[6 * (fo + s) + k];
      ((int32_t*)(rec + L.daabb))[6 * s + k] = src.daabb[6 * (fo + s) + k];
    }
    for (int k = 0; k < 4; ++k) ((int32_t*)(rec + L.bbox))[4 * s + k] = src.bbox[4 * (fo + s) + k];
  }
  if (sem)
    for (size_t i = tid; i < (size_t)S * Df; i += nt) ((float*)(rec + L.emb))[i] = src.emb[fo * Df + i];
  for (size_t i = tid; i < (size_t)S * Dt; i += nt) ((double*)(rec + L.trk))[i] = src.trk[fo * Dt + i];
}

__global__ void k_det_unpack(const uint8_t* buf, int n, int G, int nloc, DetLayout L, WinBufs dst, FrameMeta* meta_dst,
                             int Df, int Dt, int sem) {
  const int i = blockIdx.y;
  if (i >= n) return;
  const int r = i % G, j = i / G;
  const uint8_t* rec = buf + ((size_t)r * nloc + j) * L.total;
  const int64_t* mt = (const int64_t*)(rec + L.meta);
  const int S = (int)mt[0];
  const size_t fo = (size_t)i * dst.SMAX;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    meta_dst[i].S = S;
    meta_dst[i].frame_id = mt[1];
    dst.oor[i] = (unsigned long long)mt[2];
  }
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int s = tid; s < S; s += nt) {
    dst.status[fo + s] = ((const int32_t*)(rec + L.status))[s];
    dst.vs[fo + s] = ((const uint32_t*)(rec + L.vs))[s];
    dst.area[fo + s] = ((const uint32_t*)(rec + L.area))[s];
    dst.tok[fo + s] = rec[L.tok + s];
    for (int k = 0; k < 6; ++k) {
      dst.qf[6 * (fo + s) + k] = ((const float*)(rec + L.qf))[6 * s + k];
      dst.daabb[6 * (fo + s) + k] = ((const int32_t*)(rec + L.daabb))[6 * s + k];
    }
    for (int k = 0; k < 4; ++k) dst.bbox[4 * (fo + s) + k] = ((const int32_t*)(rec + L.bbox))[4 * s + k];
  }
  if (sem)
    for (size_t x = tid; x < (size_t)S * Df; x += nt) dst.emb[fo * Df + x] = ((const float*)(rec + L.emb))[x];
  for (size_t x = tid; x < (size_t)S * Dt; x += nt) dst.trk[fo * Dt + x] = ((const double*)(rec + L.trk))[x];
}

// one thread per pair of the shard's frame j (window slot g + G j); pairs of dropped detections
// stay home (stage 2 never reads them).  Mode: dst != nullptr -> direct delivery (same device);
// else counts (offsets == nullptr) or scatter into send at offsets[owner] (NCCL all-to-all).
__global__ void __launch_bounds__(256) k_pair_route(WinBufs src, int n, int g, int G, const RouteDst* dst,
                                                    unsigned long long* counts, const unsigned long long* offsets,
                                                    PairRec* send, int* err) {
  const int j = blockIdx.y;
  if (j >= n) return;
  const int slot = g + G * j;
  const uint32_t np = min(src.npairs[j], (uint32_t)src.PMAX);
  const size_t fo = (size_t)j * src.PMAX;
  const int32_t* st = src.status + (size_t)j * src.SMAX;
  __shared__ unsigned long long cnt_s[MAX_LOCAL_SHARDS * 8];
  const bool counting = dst == nullptr && offsets == nullptr;
  if (counting)
    for (int d = threadIdx.x; d < G; d += blockDim.x) cnt_s[d] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t s = src.pinfo[fo + i];
    if (st[s] != 0) continue;
    const unsigned long long key = src.pkey[fo + i];
    const uint32_t o = key_owner(key, (uint32_t)G);
    if (dst) {
      const uint32_t pos = atomicAdd(dst->npairs[o] + slot, 1u);
      if (pos < (uint32_t)dst->PMAX) {
        dst->pkey[o][(size_t)slot * dst->PMAX + pos] = key;
        dst->pinfo[o][(size_t)slot * dst->PMAX + pos] = s;
      } else {
        raise_err(err, DERR_FRAME_PAIRS);
      }
    } else if (counting) {
      atomicAdd(&cnt_s[o], 1ull);
    } else {
      const unsigned long long pos = atomicAdd(&counts[o], 1ull);   // counts reset to 0 before the scatter
      send[offsets[o] + pos] = PairRec{key, ((uint32_t)slot << 8) | s, 0u};
    }
  }
  if (counting) {
    __syncthreads();
    for (int d = threadIdx.x; d < G; d += blockDim.x)
      if (cnt_s[d]) atomicAdd(&counts[d], cnt_s[d]);
  }
}

__global__ void __launch_bounds__(256) k_pair_deliver(const PairRec* recv, unsigned long long n, WinBufs dst, int* err) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const PairRec r = recv[i];
    const uint32_t slot = r.info >> 8;
    const uint32_t pos = atomicAdd(dst.npairs + slot, 1u);
    if (pos < (uint32_t)dst.PMAX) {
      dst.pkey[(size_t)slot * dst.PMAX + pos] = r.key;
      dst.pinfo[(size_t)slot * dst.PMAX + pos] = r.info & 0xFFu;
    } else {
      raise_err(err, DERR_FRAME_PAIRS);
    }
  }
}

void launch_det_pack(const WinBufs& src, int n, const FrameMeta* meta_host, uint8_t* buf, const DetLayout& L, int Df,
                     int Dt, bool sem, cudaStream_t st) {
  if (n <= 0) return;
  MetaArr ma{};
  for (int j = 0; j < n && j < MAXWIN; ++j) ma.m[j] = meta_host[j];
  k_det_pack<<<dim3(8, n), 256, 0, st>>>(src, n, ma, buf, L, Df, Dt, sem ? 1 : 0);
  debug_check(st, "k_det_pack", -1);
}

void launch_det_unpack(const uint8_t* buf, int n, int G, int nloc, const DetLayout& L, const WinBufs& dst,
                       FrameMeta* meta_dst, int Df, int Dt, bool sem, cudaStream_t st) {
  if (n <= 0) return;
  k_det_unpack<<<dim3(8, n), 256, 0, st>>>(buf, n, G, nloc, L, dst, meta_dst, Df, Dt, sem ? 1 : 0);
  debug_check(st, "k_det_unpack", -1);
}

void launch_pair_route(const WinBufs& src, int n, int g, int G, const RouteDst* dst, unsigned long long* counts,
                       const unsigned long long* offsets, PairRec* send, int* err, cudaStream_t st) {
  if (n <= 0) return;
  k_pair_route<<<dim3(64, n), 256, 0, st>>>(src, n, g, G, dst, counts, offsets, send, err);
  debug_check(st, "k_pair_route", -1);
}

void launch_pair_deliver(const PairRec* recv, unsigned long long n, const WinBufs& dst, int* err, cudaStream_t st) {
  if (n == 0) return;
  k_pair_deliver<<<256, 256, 0, st>>>(recv, n, dst, err);
  debug_check(st, "k_pair_deliver", -1);
}

}  // namespace disc
