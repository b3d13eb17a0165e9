// k_query.cu -- off-path readers of the map: Q1 query, Q2 instance export
// and the membership export used by the parity tests.
#include <cstdio>
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

// ------------------------------------------------------------------------------------------
// NEXT row f4: batched open-vocabulary retrieval.
//  classify_topk (P:195 [§IV-A], R39): cos(e_j, t_c) = e_j . t_c / |t_c| for every live
//  instance with an embedding x every class row, the k best per instance (descending, ties by
//  ascending class index).  A dense contraction E [n x Df] x T^T [Df x C] with a per-row top-k
//  epilogue fused in: 64 x 64 output tiles from shared-memory K-slices (fp32 FFMA, 4 x 4 outputs
//  per thread), each tile's scores merged into the rows' running top-k lists in shared memory, so
//  the n x C score matrix never reaches HBM.
// ------------------------------------------------------------------------------------------
constexpr int CL_T = 64, CL_K = 32, CL_KMAX = 16;

__global__ void __launch_bounds__(256) k_classify(MapState M, int Df, const int32_t* ids, int n, const float* tab,
                                                  const double* tnorm, int C, int k, int32_t* out_c, float* out_s) {
  __shared__ float As[CL_K][CL_T + 1], Bs[CL_K][CL_T + 1];
  __shared__ float S[CL_T][CL_T + 1];
  __shared__ float tk_s[CL_T][CL_KMAX];
  __shared__ int32_t tk_c[CL_T][CL_KMAX];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.x * CL_T;
  for (int i = threadIdx.x; i < CL_T * CL_KMAX; i += blockDim.x) {
    tk_s[i / CL_KMAX][i % CL_KMAX] = -INFINITY;
    tk_c[i / CL_KMAX][i % CL_KMAX] = INT32_MAX;
  }
  for (int c0 = 0; c0 < C; c0 += CL_T) {
    float acc[4][4] = {};
    for (int d0 = 0; d0 < Df; d0 += CL_K) {
      for (int i = threadIdx.x; i < CL_K * CL_T; i += blockDim.x) {
        const int row = i / CL_K, dd = i % CL_K;   // consecutive threads: consecutive dims of one row
        const int r = r0 + row, c = c0 + row, d = d0 + dd;
        As[dd][row] = (r < n && d < Df) ? M.E[(size_t)ids[r] * Df + d] : 0.f;
        Bs[dd][row] = (c < C && d < Df) ? tab[(size_t)c * Df + d] : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int dd = 0; dd < CL_K; ++dd) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] = As[dd][ty * 4 + i]; b[i] = Bs[dd][tx * 4 + i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + tx * 4 + j;
        S[ty * 4 + i][tx * 4 + j] = c < C ? (tnorm[c] > 0.0 ? (float)((double)acc[i][j] / tnorm[c]) : 0.f) : -INFINITY;
      }
    __syncthreads();
    if (threadIdx.x < CL_T) {   // merge the tile into row threadIdx.x's top-k (classes ascending: ties keep the lower index)
      const int row = threadIdx.x;
      for (int j = 0; j < CL_T && c0 + j < C; ++j) {
        const float v = S[row][j];
        if (!(v > tk_s[row][k - 1])) continue;
        int pos = k - 1;
        while (pos > 0 && v > tk_s[row][pos - 1]) {
          tk_s[row][pos] = tk_s[row][pos - 1];
          tk_c[row][pos] = tk_c[row][pos - 1];
          --pos;
        }
        tk_s[row][pos] = v;
        tk_c[row][pos] = c0 + j;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < CL_T && r0 + threadIdx.x < n)
    for (int i = 0; i < k; ++i) {
      out_c[(size_t)(r0 + threadIdx.x) * k + i] = tk_c[threadIdx.x][i];
      out_s[(size_t)(r0 + threadIdx.x) * k + i] = tk_s[threadIdx.x][i];
    }
}

__global__ void k_table_norms(const float* tab, int C, int Df, double* tnorm) {
  const int lane = threadIdx.x & 31;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < C; c += (gridDim.x * blockDim.x) >> 5) {
    double a = 0;
    for (int d = lane; d < Df; d += 32) a += (double)tab[(size_t)c * Df + d] * tab[(size_t)c * Df + d];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) tnorm[c] = sqrt(a);
  }
}

int64_t run_classify(const MapState& M, int Df, int64_t next_id, const float* table_host, int32_t C, int32_t k,
                     int64_t* ids_out, int32_t* cls_out, float* sc_out, int64_t cap, cudaStream_t st, void* scratch,
                     size_t scratch_bytes) {
  Scratch sc{(char*)scratch, scratch_bytes};
  const int64_t nn = next_id > 0 ? next_id : 1;
  int32_t* ids = sc.take<int32_t>(nn);
  int32_t* nsel = sc.take<int32_t>(1);
  float* tab = sc.take<float>((size_t)C * Df);
  double* tnorm = sc.take<double>(C);
  if (!ids || !nsel || !tab || !tnorm) return -1;
  const int32_t n = select_ids(M, next_id, 1, ids, nsel, sc, st);
  if (n < 0) return -1;
  if (!ids_out || n == 0) return n;
  const int kk = k < C ? k : C;
  const int m = (int)(n < cap ? n : cap);
  int32_t* dc = sc.take<int32_t>((size_t)m * kk);
  float* ds = sc.take<float>((size_t)m * kk);
  if (!dc || !ds) return -1;
  cudaMemcpyAsync(tab, table_host, sizeof(float) * C * Df, cudaMemcpyHostToDevice, st);
  k_table_norms<<<64, 256, 0, st>>>(tab, C, Df, tnorm);
  k_classify<<<(m + CL_T - 1) / CL_T, 256, 0, st>>>(M, Df, ids, m, tab, tnorm, C, kk, dc, ds);
  static thread_local std::vector<int32_t> hid;
  hid.resize(m);
  cudaMemcpyAsync(hid.data(), ids, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(cls_out, dc, sizeof(int32_t) * m * kk, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(sc_out, ds, sizeof(float) * m * kk, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  for (int i = 0; i < m; ++i) ids_out[i] = hid[i];
  return n;
}

// ------------------------------------------------------------------------------------------
//  dense transfer (P:201 [§IV-B], R40): the nearest voxel centre (k + 0.5) r over all
//  instances' voxels, searched in the voxel hash over the cube of keys within d_assign of the
//  point (thread per point); squared distances in fp64, no contraction, x + y + z in that order
//  (the oracle's arithmetic, so ties and the d_assign cut are decided identically); ties -> lower id.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t q_find(const MapState& M, uint64_t key) {
  uint64_t h = mix64(key) & (M.MC - 1);
  for (uint64_t probe = 0; probe < M.MC; ++probe) {
    const unsigned long long k = __ldcg(&M.slots[h].key);
    if (k == key) return (uint32_t)h;
    if (k == KEY_EMPTY) return U32_EMPTY;
    h = (h + 1) & (M.MC - 1);
  }
  return U32_EMPTY;
}

__global__ void k_dense_transfer(MapState M, const float* pts, int64_t P, double r, int R, double dmax2, int64_t* out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const double x[3] = {(double)pts[3 * p], (double)pts[3 * p + 1], (double)pts[3 * p + 2]};
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = (int)floor(x[a] / r);
    double best = INFINITY;
    int64_t bid = -1;
    for (int dx = -R; dx <= R; ++dx)
      for (int dy = -R; dy <= R; ++dy)
        for (int dz = -R; dz <= R; ++dz) {
          const int k[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
          bool inr = true;
          for (int a = 0; a < 3; ++a) inr = inr && k[a] >= -KEY_BIAS && k[a] < KEY_BIAS;
          if (!inr) continue;
          double d2 = 0.0;
          for (int a = 0; a < 3; ++a) {
            const double ce = __dmul_rn(__dadd_rn((double)k[a], 0.5), r);
            const double t = __dsub_rn(x[a], ce);
            d2 = __dadd_rn(d2, __dmul_rn(t, t));
          }
          if (d2 > dmax2 || d2 > best) continue;
          const uint64_t key = ((uint64_t)(uint32_t)(k[0] + KEY_BIAS) << 42) |
                               ((uint64_t)(uint32_t)(k[1] + KEY_BIAS) << 21) | (uint64_t)(uint32_t)(k[2] + KEY_BIAS);
          const uint32_t h = q_find(M, key);
          if (h == U32_EMPTY) continue;
          const uint32_t* labs = M.slots[h].lab;
          int nl = INLINE_LABELS;
          uint32_t nx = M.slots[h].ovf;
          bool done = false;
          while (!done) {
            for (int i = 0; i < nl; ++i) {
              const uint32_t L = labs[i];
              if (L == U32_EMPTY) { done = true; break; }
              if (L == LAB_TOMB) continue;
              const int64_t id = M.id_of[L];
              if (d2 < best || (d2 == best && id < bid)) { best = d2; bid = id; }
            }
            if (done || nx == U32_EMPTY) break;
            labs = M.ovf[nx].lab;
            nl = CHUNK_LABELS;
            nx = M.ovf[nx].next;
          }
        }
    out[p] = bid;
  }
}

int run_dense_transfer(const MapState& M, float r, const float* pts_host, int64_t P, float d_assign, int64_t* out_host,
                       cudaStream_t st, void* scratch, size_t scratch_bytes) {
  Scratch sc{(char*)scratch, scratch_bytes};
  float* pts = sc.take<float>((size_t)P * 3);
  int64_t* out = sc.take<int64_t>((size_t)P);
  if (!pts || !out) return -1;
  const double rd = (double)r, dd = (double)d_assign;
  const int R = (int)ceil(dd / rd) + 1;
  cudaMemcpyAsync(pts, pts_host, sizeof(float) * 3 * P, cudaMemcpyHostToDevice, st);
  k_dense_transfer<<<(int)std::min<int64_t>((P + 127) / 128, 4096), 128, 0, st>>>(M, pts, P, rd, R, dd * dd, out);
  cudaMemcpyAsync(out_host, out, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return 0;
}

// Diagnostic (DISC_SLOT_STATS, printed by disc_get_stats): label-list shape over the voxel hash --
// keys, live labels, tombstones, keys with overflow chunks, chunks on the longest list.
__global__ void k_slot_stats(MapState M, unsigned long long* out) {
  unsigned long long keys = 0, live = 0, tomb = 0, ovf = 0, maxch = 0;
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < M.MC; h += (uint64_t)gridDim.x * blockDim.x) {
    const KeySlot& ks = M.slots[h];
    if (ks.key == KEY_EMPTY) continue;
    ++keys;
    for (int i = 0; i < INLINE_LABELS; ++i) {
      if (ks.lab[i] == U32_EMPTY) break;
      if (ks.lab[i] == LAB_TOMB) ++tomb; else ++live;
    }
    unsigned long long ch = 0;
    for (uint32_t nx = ks.ovf; nx != U32_EMPTY; nx = M.ovf[nx].next) {
      ++ch;
      for (int i = 0; i < CHUNK_LABELS; ++i) {
        const uint32_t L = M.ovf[nx].lab[i];
        if (L == U32_EMPTY) break;
        if (L == LAB_TOMB) ++tomb; else ++live;
      }
    }
    if (ch) ++ovf;
    maxch = max(maxch, ch);
  }
  atomicAdd(&out[0], keys); atomicAdd(&out[1], live); atomicAdd(&out[2], tomb); atomicAdd(&out[3], ovf);
  atomicMax(&out[4], maxch);
}

void slot_stats(const MapState& M, cudaStream_t st) {
  unsigned long long* d = nullptr;
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  if (cudaMalloc(&d, sizeof(h)) != cudaSuccess) return;
  cudaMemsetAsync(d, 0, sizeof(h), st);
  k_slot_stats<<<1024, 256, 0, st>>>(M, d);
  cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  fprintf(stderr, "slot stats: keys %llu live labels %llu tombstones %llu keys with overflow chunks %llu longest chain %llu\n",
          h[0], h[1], h[2], h[3], h[4]);
}

}  // namespace disc
