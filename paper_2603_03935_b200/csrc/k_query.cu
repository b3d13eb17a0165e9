// k_query.cu -- off-path readers of the map: Q1 query, Q2 instance export
// and the membership export used by the parity tests.
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "disc_common.cuh"
#include "disc_launch.h"

namespace disc {

__global__ void k_alive_flags(MapState M, int64_t n, uint8_t* flags, int want_embed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = M.alive[i] && (!want_embed || M.q[i] >= 0.f) ? 1 : 0;
}

__global__ void k_gather_instances(MapState M, int Df, int Dt, const int32_t* ids, const int32_t* nsel,
                                   int32_t cap, disc_instance* out, float* emb, double* trk) {
  const int n = min(*nsel, cap);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int id = ids[i];
    if (threadIdx.x == 0) {
      disc_instance r;
      r.id = id;
      r.voxel_count = M.vcount[id];
      r.last_seen = M.last_seen[id];
      r.obs_count = M.obs[id];
      r.q = M.q[id];
      for (int k = 0; k < 3; ++k) {
        r.aabb_min[k] = M.aabb[(size_t)id * 6 + k];
        r.aabb_max[k] = M.aabb[(size_t)id * 6 + 3 + k];
      }
      out[i] = r;
    }
    if (emb)
      for (int d = threadIdx.x; d < Df; d += blockDim.x) emb[(size_t)i * Df + d] = M.E[(size_t)id * Df + d];
    if (trk)
      for (int d = threadIdx.x; d < Dt; d += blockDim.x) trk[(size_t)i * Dt + d] = M.T[(size_t)id * Dt + d];
  }
}

struct Scratch {   // bump allocator over a caller-provided device buffer
  char* p;
  size_t left;
  template <typename T>
  T* take(size_t n) {
    const size_t b = (n * sizeof(T) + 255) & ~(size_t)255;
    if (b > left) return nullptr;
    T* r = (T*)p;
    p += b;
    left -= b;
    return r;
  }
};

static int32_t select_ids(const MapState& M, int64_t n, int want_embed, int32_t* ids, int32_t* nsel,
                          Scratch& sc, cudaStream_t st) {
  uint8_t* flags = sc.take<uint8_t>(n > 0 ? n : 1);
  if (!flags) return -1;
  k_alive_flags<<<256, 256, 0, st>>>(M, n, flags, want_embed);
  size_t tb = 0;
  thrust::counting_iterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb, it, flags, ids, nsel, (int)n, st);
  void* tmp = sc.take<char>(tb);
  if (!tmp) return -1;
  cub::DeviceSelect::Flagged(tmp, tb, it, flags, ids, nsel, (int)n, st);
  int32_t h = 0;
  cudaMemcpyAsync(&h, nsel, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}

int64_t export_instances(const MapState& M, int Df, int Dt, int64_t next_id, disc_instance* out, float* embeds,
                         double* track, int32_t cap, cudaStream_t st, void* scratch, size_t scratch_bytes) {
  Scratch sc{(char*)scratch, scratch_bytes};
  int32_t* ids = sc.take<int32_t>(next_id > 0 ? next_id : 1);
  int32_t* nsel = sc.take<int32_t>(1);
  if (!ids || !nsel) return -1;
  const int32_t n = select_ids(M, next_id, 0, ids, nsel, sc, st);
  if (n < 0 || !out || n == 0) return n;
  const int32_t m = n < cap ? n : cap;
  disc_instance* d_out = sc.take<disc_instance>(m);
  float* d_emb = embeds ? sc.take<float>((size_t)m * Df) : nullptr;
  double* d_trk = (track && Dt > 0) ? sc.take<double>((size_t)m * Dt) : nullptr;
  if (!d_out || (embeds && !d_emb) || (track && Dt > 0 && !d_trk)) return -1;
  k_gather_instances<<<256, 128, 0, st>>>(M, Df, Dt, ids, nsel, m, d_out, d_emb, d_trk);
  cudaMemcpyAsync(out, d_out, sizeof(disc_instance) * m, cudaMemcpyDeviceToHost, st);
  if (embeds) cudaMemcpyAsync(embeds, d_emb, sizeof(float) * m * Df, cudaMemcpyDeviceToHost, st);
  if (d_trk) cudaMemcpyAsync(track, d_trk, sizeof(double) * m * Dt, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return n;
}

__global__ void k_memberships(MapState M, unsigned long long* keys, int64_t* ids, unsigned long long cap,
                              unsigned long long* n) {
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < M.MC; h += (uint64_t)gridDim.x * blockDim.x) {
    const KeySlot& ks = M.slots[h];
    if (ks.key == KEY_EMPTY) continue;
    const uint32_t* labs = ks.lab;
    int nl = INLINE_LABELS;
    uint32_t nx = ks.ovf;
    while (true) {
      for (int i = 0; i < nl; ++i) {
        const uint32_t L = labs[i];
        if (L == U32_EMPTY) break;
        if (L == LAB_TOMB) continue;
        const unsigned long long w = atomicAdd(n, 1ull);
        if (w < cap) {
          keys[w] = ks.key;
          ids[w] = M.id_of[L];
        }
      }
      if (nx == U32_EMPTY) break;
      labs = M.ovf[nx].lab;
      nl = CHUNK_LABELS;
      nx = M.ovf[nx].next;
    }
  }
}

int64_t export_memberships(const MapState& M, uint64_t* keys, int64_t* ids, int64_t cap, cudaStream_t st,
                           void* scratch, size_t scratch_bytes) {
  Scratch sc{(char*)scratch, scratch_bytes};
  unsigned long long* n = sc.take<unsigned long long>(1);
  const int64_t room = keys ? cap : 0;
  unsigned long long* dk = room ? sc.take<unsigned long long>(room) : nullptr;
  int64_t* di = room ? sc.take<int64_t>(room) : nullptr;
  if (!n || (room && (!dk || !di))) return -1;
  cudaMemsetAsync(n, 0, sizeof(unsigned long long), st);
  k_memberships<<<1024, 256, 0, st>>>(M, dk, di, (unsigned long long)room, n);
  unsigned long long hn = 0;
  cudaMemcpyAsync(&hn, n, sizeof(hn), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (room && hn <= (unsigned long long)cap) {
    cudaMemcpyAsync(keys, dk, sizeof(uint64_t) * hn, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(ids, di, sizeof(int64_t) * hn, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  }
  return (int64_t)hn;
}

// score_j = e_j . q / |q|: one warp per selected instance
__global__ void k_scores(MapState M, int Df, const float* q, const int32_t* ids, const int32_t* nsel, float* sc) {
  const int n = *nsel;
  const int lane = threadIdx.x & 31;
  double qq = 0;
  for (int d = lane; d < Df; d += 32) qq += (double)q[d] * q[d];
#pragma unroll
  for (int o = 16; o; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  const double qn = sqrt(qq);
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const float* e = M.E + (size_t)ids[i] * Df;
    double a = 0;
    for (int d = lane; d < Df; d += 32) a += (double)e[d] * ((double)q[d] / qn);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sc[i] = (float)a;
  }
}

int32_t run_query(const MapState& M, int Df, int64_t next_id, const float* q_host, int32_t k, int64_t* ids_out,
                  float* scores_out, cudaStream_t st, void* scratch, size_t scratch_bytes) {
  Scratch sc{(char*)scratch, scratch_bytes};
  const int64_t nn = next_id > 0 ? next_id : 1;
  int32_t* ids = sc.take<int32_t>(nn);
  int32_t* nsel = sc.take<int32_t>(1);
  float* q = sc.take<float>(Df);
  float* score = sc.take<float>(nn);
  float* score2 = sc.take<float>(nn);
  int32_t* ids2 = sc.take<int32_t>(nn);
  if (!ids || !nsel || !q || !score || !score2 || !ids2) return -1;
  cudaMemcpyAsync(q, q_host, sizeof(float) * Df, cudaMemcpyHostToDevice, st);
  const int32_t n = select_ids(M, next_id, 1, ids, nsel, sc, st);
  if (n <= 0) return n;
  k_scores<<<256, 256, 0, st>>>(M, Df, q, ids, nsel, score);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, score, score2, ids, ids2, n, 0, 32, st);
  void* tmp = sc.take<char>(tb);
  if (!tmp) return -1;
  // radix sort is stable: equal scores keep ascending id order
  cub::DeviceRadixSort::SortPairsDescending(tmp, tb, score, score2, ids, ids2, n, 0, 32, st);
  const int32_t m = n < k ? n : k;
  static thread_local std::vector<int32_t> hid;
  hid.resize(m);
  cudaMemcpyAsync(scores_out, score2, sizeof(float) * m, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hid.data(), ids2, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  for (int i = 0; i < m; ++i) ids_out[i] = hid[i];
  return m;
}

}  // namespace disc
