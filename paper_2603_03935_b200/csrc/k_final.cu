// k_final.cu -- disc_finalize: P:100 [§III-B] "a final, lightweight
// post-processing step iterates over the map to merge remaining orphaned candidates and filter out
// residual noisy instances, such as segments containing fewer than a minimum threshold of voxels";
// S:333-337.  Readings R35-R38, the same as oracle/ora_finalize:
//  R35 rounds of snapshot union-find over instance pairs until no pair qualifies;
//  R36 pair test c_ij >= 1 and c_ij >= tau_geo min(|V_i|, |V_j|) (exact fp64), gate
//      (dot_pin(T_i,T_j) / sqrt(TT_i)) / sqrt(TT_j) >= tau_vis (i < j), zero norm -> -2;
//  R37 merge into the min id: T summed in ascending id order, (e, Q) replaced in ascending order iff
//      strictly higher, obs summed, last_seen = max, V = union (labels remapped in place);
//  R38 the minimum-size filter after the fixpoint.
// Once per run (not the per-frame path): whole-map passes over the voxel hash are fine here.
//
//  F1 k_fin_pairs    every key with >= 2 labels adds 1 to each of its (id_i < id_j) pairs
//  F2 k_fin_edges    warp per pair: R36 test; a qualifying pair links i and j in a lock-free
//                    union-find whose root is always the smaller id
//  F3 k_fin_members  members of non-trivial components as (root << 32 | id) keys, CUB-sorted
//  F4 k_fin_merge    warp per component: R37 in ascending id order; label remap old -> root's
//  F5 k_fin_relabel  every key's labels remapped (or dropped, R38) and deduplicated in place;
//                    |V| and the key-space AABB recounted exactly from the keys
//  F6 k_fin_lists    per-label key lists rebuilt from the keys (exclusive scan of |V|)
#include <cub/cub.cuh>

#include "disc_common.cuh"
#include "disc_launch.h"

namespace disc {

constexpr uint32_t LAB_DROP = 0xFFFFFFFDu;   // remap target: label removed (R38)
constexpr int FIN_MAXL = 64;                   // labels per key handled in local memory

struct FinBufs {
  unsigned long long* pkey;   // [PC] pair table codes (i << 32 | j)
  uint32_t* pcnt;             // [PC]
  uint32_t PC;                // power of two
  uint32_t* par;              // [IMAX] union-find parent (ids)
  uint32_t* remap;            // [IMAX] physical label -> new label (U32_EMPTY = unchanged)
  uint32_t* flag;             // [IMAX] component has members / scratch
  unsigned long long* keys;   // [IMAX] (root << 32 | id) of members, then sorted copy
  unsigned long long* keys2;
  uint32_t* nkeys;            // [1]
  unsigned long long* rep;    // [8]: edges, merged_away, relabeled, removed, live_inst, live_mem
  int* err;
};

// the live (non-tombstone) physical labels of slot h, in list order
__device__ int fin_labels(const MapState& M, uint64_t h, uint32_t* out, bool* over) {
  int n = 0;
  const KeySlot& S = M.slots[h];
  for (int i = 0; i < INLINE_LABELS; ++i) {
    const uint32_t L = S.lab[i];
    if (L == U32_EMPTY) return n;
    if (L == LAB_TOMB) continue;
    if (n < FIN_MAXL) out[n++] = L; else *over = true;
  }
  for (uint32_t nx = S.ovf; nx != U32_EMPTY; nx = M.ovf[nx].next) {
    for (int i = 0; i < CHUNK_LABELS; ++i) {
      const uint32_t L = M.ovf[nx].lab[i];
      if (L == U32_EMPTY) return n;
      if (L == LAB_TOMB) continue;
      if (n < FIN_MAXL) out[n++] = L; else *over = true;
    }
  }
  return n;
}

__device__ __forceinline__ void fin_pair_add(const FinBufs& B, unsigned long long code) {
  uint32_t h = (uint32_t)mix64(code) & (B.PC - 1);
  for (uint32_t probe = 0; probe < B.PC; ++probe) {
    unsigned long long k = __ldcg(&B.pkey[h]);
    if (k == KEY_EMPTY) {
      k = atomicCAS(&B.pkey[h], KEY_EMPTY, code);
      if (k == KEY_EMPTY) k = code;
    }
    if (k == code) {
      atomicAdd(&B.pcnt[h], 1u);
      return;
    }
    h = (h + 1) & (B.PC - 1);
  }
  raise_err(B.err, DERR_TRIPLES);
}

__global__ void __launch_bounds__(256) k_fin_pairs(MapState M, FinBufs B) {
  uint32_t lab[FIN_MAXL], ids[FIN_MAXL];
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < M.MC; h += (uint64_t)gridDim.x * blockDim.x) {
    if (M.slots[h].key == KEY_EMPTY || M.slots[h].lab[1] == U32_EMPTY) continue;   // < 2 label cells
    bool over = false;
    const int n = fin_labels(M, h, lab, &over);
    if (over) raise_err(B.err, 1000 + __LINE__);
    for (int i = 0; i < n; ++i) {   // ids ascending (insertion sort; a handful per key)
      const uint32_t v = M.id_of[lab[i]];
      int k = i;
      while (k > 0 && ids[k - 1] > v) { ids[k] = ids[k - 1]; --k; }
      ids[k] = v;
    }
    for (int a = 0; a < n; ++a)
      for (int b = a + 1; b < n; ++b)
        if (ids[a] != ids[b]) fin_pair_add(B, ((unsigned long long)ids[a] << 32) | ids[b]);
  }
}

__device__ uint32_t uf_find(uint32_t* par, uint32_t x) {
  while (true) {
    const uint32_t p = __ldcg(&par[x]);
    if (p == x) return x;
    const uint32_t gp = __ldcg(&par[p]);
    if (gp != p) atomicCAS(&par[x], p, gp);   // path halving
    x = p;
  }
}

__device__ void uf_union(uint32_t* par, uint32_t a, uint32_t b) {
  while (true) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    if (a == b) return;
    if (a > b) { const uint32_t t = a; a = b; b = t; }
    if (atomicCAS(&par[b], b, a) == b) return;   // the larger root under the smaller: root = min id
  }
}

__global__ void __launch_bounds__(256) k_fin_edges(MapState M, FinBufs B, float tau_geo, float tau_vis, int Dt) {
  const int lane = threadIdx.x & 31;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = w0; e < B.PC; e += nw) {
    const unsigned long long code = B.pkey[e];
    if (code == KEY_EMPTY) continue;
    const uint32_t c = B.pcnt[e];
    const uint32_t i = (uint32_t)(code >> 32), j = (uint32_t)code;
    const int64_t mn = min(M.vcount[i], M.vcount[j]);
    bool ok = c >= 1 && (double)c >= (double)tau_geo * (double)mn;   // R36 (R10's exact test)
    if (ok && Dt > 0) {
      const double ti = M.TT[i], tj = M.TT[j];
      const double d = dot_pin_reg(M.T + (size_t)i * Dt, M.T + (size_t)j * Dt, Dt);
      double cosv = -2.0;
      if (ti > 0.0 && tj > 0.0) cosv = __ddiv_rn(__ddiv_rn(d, __dsqrt_rn(ti)), __dsqrt_rn(tj));
      ok = cosv >= (double)tau_vis;
    }
    if (lane == 0) {
      if (ok) {
        atomicAdd(&B.rep[0], 1ull);
        uf_union(B.par, i, j);
      }
      B.pkey[e] = KEY_EMPTY;   // the table is empty again for the next round
      B.pcnt[e] = 0;
    }
    __syncwarp();
  }
}

// members of non-trivial components: (root << 32 | id), the root itself included
__global__ void k_fin_members(MapState M, FinBufs B, uint32_t n) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
    if (!M.alive[id]) continue;
    const uint32_t r = uf_find(B.par, id);
    if (r != id) {
      B.keys[atomicAdd(B.nkeys, 1u)] = ((unsigned long long)r << 32) | id;
      if (atomicExch(&B.flag[r], 1u) == 0u) B.keys[atomicAdd(B.nkeys, 1u)] = ((unsigned long long)r << 32) | r;
    }
  }
}

// warp per component (sorted keys: the root first, then its members ascending)
__global__ void __launch_bounds__(256) k_fin_merge(MapState M, FinBufs B, const unsigned long long* sk, uint32_t nk,
                                                   int Df, int Dt) {
  const int lane = threadIdx.x & 31;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t s0 = w0; s0 < nk; s0 += nw) {
    const uint32_t r = (uint32_t)(sk[s0] >> 32);
    if (s0 > 0 && (uint32_t)(sk[s0 - 1] >> 32) == r) continue;   // not a component's first entry
    uint32_t e = s0 + 1;
    while (e < nk && (uint32_t)(sk[e] >> 32) == r) ++e;
    // T: ((T_r + T_m1) + T_m2) ..., elementwise fp64, ascending ids (R37)
    for (int d = lane; d < Dt; d += 32) {
      double acc = M.T[(size_t)r * Dt + d];
      for (uint32_t k = s0 + 1; k < e; ++k) acc = __dadd_rn(acc, M.T[(size_t)(uint32_t)sk[k] * Dt + d]);
      M.T[(size_t)r * Dt + d] = acc;
    }
    __syncwarp();
    if (Dt > 0) {
      const double tt = dot_pin_reg(M.T + (size_t)r * Dt, M.T + (size_t)r * Dt, Dt);
      if (lane == 0) M.TT[r] = tt;
    }
    // (e, Q): the root's, replaced in ascending order iff strictly higher
    float q = M.q[r];
    uint32_t src = r;
    int obs = M.obs[r];
    int64_t ls = M.last_seen[r];
    unsigned long long rel = 0;
    for (uint32_t k = s0 + 1; k < e; ++k) {
      const uint32_t mid = (uint32_t)sk[k];
      const float qm = M.q[mid];
      if (qm > q) { q = qm; src = mid; }
      obs += M.obs[mid];
      ls = max(ls, M.last_seen[mid]);
      rel += (unsigned long long)M.vcount[mid];
    }
    if (src != r)
      for (int d = lane; d < Df; d += 32) M.E[(size_t)r * Df + d] = M.E[(size_t)src * Df + d];
    const uint32_t Lr = M.phys_of[r];
    for (uint32_t k = s0 + 1 + lane; k < e; k += 32) {
      const uint32_t mid = (uint32_t)sk[k];
      B.remap[M.phys_of[mid]] = Lr;
      M.alive[mid] = 0;
      M.phys_of[mid] = U32_EMPTY;
    }
    if (lane == 0) {
      M.q[r] = q;
      M.obs[r] = obs;
      M.last_seen[r] = ls;
      atomicAdd(&B.rep[1], (unsigned long long)(e - s0 - 1));
      atomicAdd(&B.rep[2], rel);
    }
  }
}

__global__ void k_fin_zero(MapState M, uint32_t n) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
    if (!M.alive[id]) continue;
    M.vcount[id] = 0;
    for (int k = 0; k < 3; ++k) {
      M.aabb[(size_t)id * 6 + k] = INT32_MAX;
      M.aabb[(size_t)id * 6 + 3 + k] = INT32_MIN;
    }
  }
}

// every key: labels remapped (merged -> root's label, dropped -> gone), deduplicated, written back
// compactly (inline cells, then the chunk chain; the rest EMPTY); |V| and AABB recounted
__global__ void __launch_bounds__(256) k_fin_relabel(MapState M, FinBufs B) {
  uint32_t lab[FIN_MAXL];
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < M.MC; h += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = M.slots[h].key;
    if (key == KEY_EMPTY) continue;
    bool over = false;
    const int n0 = fin_labels(M, h, lab, &over);
    if (over) raise_err(B.err, 1000 + __LINE__);
    int n = 0;
    for (int i = 0; i < n0; ++i) {
      uint32_t L = lab[i];
      const uint32_t t = B.remap[L];
      if (t == LAB_DROP) continue;
      if (t != U32_EMPTY) L = t;
      bool dup = false;
      for (int k = 0; k < n; ++k) dup = dup || lab[k] == L;
      if (!dup) lab[n++] = L;
    }
    // write back
    KeySlot& S = M.slots[h];
    int w = 0;
    for (int i = 0; i < INLINE_LABELS; ++i) S.lab[i] = w < n ? lab[w++] : U32_EMPTY;
    for (uint32_t nx = S.ovf; nx != U32_EMPTY; nx = M.ovf[nx].next)
      for (int i = 0; i < CHUNK_LABELS; ++i) M.ovf[nx].lab[i] = w < n ? lab[w++] : U32_EMPTY;
    int k3[3];
    unpack_key(key, k3[0], k3[1], k3[2]);
    for (int i = 0; i < n; ++i) {
      const uint32_t id = M.id_of[lab[i]];
      atomicAdd((unsigned long long*)&M.vcount[id], 1ull);
      for (int a = 0; a < 3; ++a) {
        atomicMin(&M.aabb[(size_t)id * 6 + a], k3[a]);
        atomicMax(&M.aabb[(size_t)id * 6 + 3 + a], k3[a]);
      }
    }
  }
}

// after a round: the merged labels' remap entries and the component flags back to "none"
__global__ void k_fin_reset(FinBufs B, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    B.remap[i] = U32_EMPTY;
    B.flag[i] = 0;
    B.par[i] = i;
  }
}

// R38: instances below min_voxels lose their labels (remap -> DROP) and die
__global__ void k_fin_filter(MapState M, FinBufs B, uint32_t n, int64_t min_voxels) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
    if (!M.alive[id] || M.vcount[id] >= min_voxels) continue;
    B.remap[M.phys_of[id]] = LAB_DROP;
    M.alive[id] = 0;
    M.phys_of[id] = U32_EMPTY;
    atomicAdd(&B.rep[3], 1ull);
  }
}

// key lists: offsets = exclusive scan of |V| over the live ids (computed by the caller), lengths
// refilled from the keys
__global__ void k_fin_list_init(MapState M, const unsigned long long* off, uint32_t n, FinBufs B) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
    const uint32_t L = M.phys_of[id];
    if (!M.alive[id]) continue;
    M.lst_off[L] = off[id];
    M.lst_cap[L] = (uint32_t)M.vcount[id];
    M.lst_len[L] = 0;
    atomicAdd(&B.rep[4], 1ull);
    atomicAdd(&B.rep[5], (unsigned long long)M.vcount[id]);
  }
}

__global__ void __launch_bounds__(256) k_fin_list_fill(MapState M) {
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < M.MC; h += (uint64_t)gridDim.x * blockDim.x) {
    if (M.slots[h].key == KEY_EMPTY) continue;
    const KeySlot& S = M.slots[h];
    auto put = [&](uint32_t L) {
      const uint32_t pos = atomicAdd(&M.lst_len[L], 1u);
      M.arena[M.lst_off[L] + pos] = (uint32_t)h;
    };
    bool done = false;
    for (int i = 0; i < INLINE_LABELS && !done; ++i) {
      if (S.lab[i] == U32_EMPTY) done = true;
      else if (S.lab[i] != LAB_TOMB) put(S.lab[i]);
    }
    for (uint32_t nx = S.ovf; nx != U32_EMPTY && !done; nx = M.ovf[nx].next)
      for (int i = 0; i < CHUNK_LABELS && !done; ++i) {
        const uint32_t L = M.ovf[nx].lab[i];
        if (L == U32_EMPTY) done = true;
        else if (L != LAB_TOMB) put(L);
      }
  }
}

__global__ void k_fin_vcount_of(MapState M, uint32_t n, unsigned long long* v) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x)
    v[id] = M.alive[id] ? (unsigned long long)M.vcount[id] : 0ull;
}

__global__ void k_fin_counters(MapState M, FinBufs B) {
  M.counters[1] = (int64_t)B.rep[4];
  M.counters[2] = (int64_t)B.rep[5];
}

// Host driver.  rep_out[7] = rounds, edges, merged_away, relabeled, removed, live_instances,
// live_memberships.  Returns 0, or -1 when a temporary allocation fails.
int run_finalize(const MapState& M, int Df, int Dt, int64_t next_id, float tau_geo, float tau_vis, int64_t min_voxels,
                 int* err, cudaStream_t st, int64_t rep_out[7]) {
  const uint32_t n = (uint32_t)std::max<int64_t>(next_id, 1);
  FinBufs B{};
  B.PC = 1u << 16;
  while (B.PC < 8u * n && B.PC < (1u << 26)) B.PC <<= 1;
  B.err = err;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n,
                                 0, 64, st);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n,
                                st);
  tmp_bytes = std::max(tmp_bytes, scan_bytes);
  void* tmp = nullptr;
  bool ok = true;
  auto alloc = [&](void** p, size_t b) { ok = ok && cudaMalloc(p, std::max<size_t>(b, 16)) == cudaSuccess; };
  alloc((void**)&B.pkey, (size_t)B.PC * 8);
  alloc((void**)&B.pcnt, (size_t)B.PC * 4);
  alloc((void**)&B.par, (size_t)n * 4);
  alloc((void**)&B.remap, (size_t)n * 4);
  alloc((void**)&B.flag, (size_t)n * 4);
  alloc((void**)&B.keys, (size_t)n * 8);
  alloc((void**)&B.keys2, (size_t)n * 8);
  alloc((void**)&B.nkeys, 4);
  alloc((void**)&B.rep, 64);
  alloc(&tmp, tmp_bytes);
  if (ok) {
    cudaMemsetAsync(B.pkey, 0xFF, (size_t)B.PC * 8, st);
    cudaMemsetAsync(B.pcnt, 0, (size_t)B.PC * 4, st);
    cudaMemsetAsync(B.rep, 0, 64, st);
    k_fin_reset<<<256, 256, 0, st>>>(B, n);
    const int G = 4 * 148;
    int64_t rounds = 0;
    for (;;) {
      unsigned long long e0 = 0, e1 = 0;
      cudaMemcpyAsync(&e0, B.rep, 8, cudaMemcpyDeviceToHost, st);
      k_fin_pairs<<<G, 256, 0, st>>>(M, B);
      k_fin_edges<<<G, 256, 0, st>>>(M, B, tau_geo, tau_vis, Dt);
      cudaMemcpyAsync(&e1, B.rep, 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (e1 == e0) break;   // fixpoint (R35)
      ++rounds;
      cudaMemsetAsync(B.nkeys, 0, 4, st);
      k_fin_members<<<256, 256, 0, st>>>(M, B, n);
      uint32_t nk = 0;
      cudaMemcpyAsync(&nk, B.nkeys, 4, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, B.keys, B.keys2, (int)nk, 0, 64, st);
      k_fin_merge<<<G, 256, 0, st>>>(M, B, B.keys2, nk, Df, Dt);
      k_fin_zero<<<256, 256, 0, st>>>(M, n);
      k_fin_relabel<<<G, 256, 0, st>>>(M, B);
      k_fin_reset<<<256, 256, 0, st>>>(B, n);
    }
    k_fin_filter<<<256, 256, 0, st>>>(M, B, n, min_voxels);
    k_fin_zero<<<256, 256, 0, st>>>(M, n);
    k_fin_relabel<<<G, 256, 0, st>>>(M, B);
    // key lists rebuilt from the keys: offsets = exclusive scan of |V| over ids
    k_fin_vcount_of<<<256, 256, 0, st>>>(M, n, B.keys);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, B.keys, B.keys2, (int)n, st);
    k_fin_list_init<<<256, 256, 0, st>>>(M, B.keys2, n, B);
    k_fin_list_fill<<<G, 256, 0, st>>>(M);
    unsigned long long hrep[8];
    cudaMemcpyAsync(hrep, B.rep, 64, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    k_fin_counters<<<1, 1, 0, st>>>(M, B);
    const unsigned long long top = hrep[5];
    cudaMemcpyAsync(M.arena_top, &top, 8, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    rep_out[0] = rounds;
    rep_out[1] = (int64_t)hrep[0];
    rep_out[2] = (int64_t)hrep[1];
    rep_out[3] = (int64_t)hrep[2];
    rep_out[4] = (int64_t)hrep[3];
    rep_out[5] = (int64_t)hrep[4];
    rep_out[6] = (int64_t)hrep[5];
  }
  for (void* p : {(void*)B.pkey, (void*)B.pcnt, (void*)B.par, (void*)B.remap, (void*)B.flag, (void*)B.keys,
                  (void*)B.keys2, (void*)B.nkeys, (void*)B.rep, tmp})
    if (p) cudaFree(p);
  return ok ? 0 : -1;
}

}  // namespace disc
