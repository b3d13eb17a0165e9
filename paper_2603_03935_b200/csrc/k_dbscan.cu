// k_dbscan.cu -- NEXT row f3: DBSCAN denoise of each segment's points before voxelisation.
// P:92 [§III-A] "The depth data corresponding to each valid segment is then projected into a 3D point
// cloud, filtered using a custom, parallelized CUDA implementation of the DBSCAN algorithm to remove
// noise, and subsequently voxelized"; only the largest cluster (by point count) is kept and
// the labels equal the classic sequential DBSCAN's.  Reading R42.
//
// The sequential algorithm, scanning a segment's points in pixel order, numbers its clusters by their
// lowest core point and gives a border point to the first cluster that reaches it.  Equivalently
// (tests/test_oracle_dbscan.py checks the equivalence on 100 random clouds): core = at least min_pts
// points within eps, the point itself included; clusters = connected components of the core points
// under "within eps", named by their lowest pixel index; a border point joins the adjacent cluster
// with the lowest name.  That form is data-parallel:
//  D1 k_db_points   (mask, point) records of every depth-valid, key-in-range masked pixel, keyed by
//                   (mask, grid cell of side 1.01 eps) -- also key_out_of_range, as K1b counts it
//  D2 CUB segmented radix sort of the records per frame (cells of one mask contiguous)
//  D3 k_db_gather   the pinned R5 world point of each sorted record
//  D4 k_db_core     neighbours within eps in the 27 adjacent cells (binary search of the sorted keys)
//  D5 k_db_union    core-core pairs within eps linked in a lock-free union-find whose root is the
//                   record with the lowest pixel index
//  D6 k_db_label    core -> its root; border -> the adjacent root with the lowest pixel; cluster sizes
//  D7 k_db_best     per mask the largest cluster (ties: the lowest root pixel = created first)
//  D8 k_db_emit     the kept points' (mask, key) pairs and normal sums into the frame tables, as K1c
// Distances are fp64 squares of the fp32 world-point differences, x + y + z, against (double)eps^2
// (no contraction): the oracle's arithmetic, so the core / border decisions match bit for bit.
#include <cub/cub.cuh>

#include "disc_common.cuh"
#include "disc_launch.h"
#include "k_stage1.cuh"

namespace disc {

constexpr int DB_CB = 18;   // bits per cell coordinate
constexpr int DB_BIAS = 1 << (DB_CB - 1);

__device__ __forceinline__ uint64_t db_cell_key(uint32_t s, int cx, int cy, int cz) {
  auto c = [](int v) { return (uint64_t)(uint32_t)(min(max(v, -DB_BIAS), DB_BIAS - 1) + DB_BIAS); };
  return ((uint64_t)s << 56) | (c(cx) << (2 * DB_CB)) | (c(cy) << DB_CB) | c(cz);
}

__device__ __forceinline__ bool db_point(const FrameDesc& F, const Params& P, int u, int v, float p[3]) {
  const float d = F.depth[(size_t)v * F.W + u];
  if (!depth_valid(d, P)) return false;
  const float xa = __fdiv_rn(__fsub_rn((float)u, F.cx), F.fx);   // R5, as K1b
  const float yb = __fdiv_rn(__fsub_rn((float)v, F.cy), F.fy);
  world_point(F, xa, yb, d, p);
  return true;
}

__device__ __forceinline__ double db_d2(const float4& a, const float4& b) {
  const double x = __dsub_rn((double)a.x, (double)b.x), y = __dsub_rn((double)a.y, (double)b.y),
               z = __dsub_rn((double)a.z, (double)b.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
}

// D1: one thread per pixel of frame blockIdx.y; the masks containing it from the mask planes
__global__ void __launch_bounds__(256) k_db_points(WinDesc wd, WinBufs wb, Params P, int* err) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int64_t HW = (int64_t)F.H * F.W;
  const float rinv = 1.0f / P.r, cinv = 1.0f / (1.01f * P.db_eps);
  uint32_t oor = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW; i += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(i % F.W), v = (int)(i / F.W);
    float p[3];
    if (!db_point(F, P, u, v, p)) continue;
    uint64_t key;
    if (!point_key_fast(p, P.r, rinv, key)) { ++oor; continue; }
    const int cx = (int)floorf(p[0] * cinv), cy = (int)floorf(p[1] * cinv), cz = (int)floorf(p[2] * cinv);
    for (int s = 0; s < F.S; ++s) {
      if (!mask_at(F, s, (size_t)i)) continue;
      const uint32_t slot = atomicAdd(&wb.dbn[f], 1u);
      if (slot >= (uint32_t)wb.DBP) { raise_err(err, DERR_FRAME_PAIRS); continue; }
      wb.dbk[(size_t)f * wb.DBP + slot] = db_cell_key((uint32_t)s, cx, cy, cz);
      wb.dbv[(size_t)f * wb.DBP + slot] = (uint32_t)i;
    }
  }
  if (oor) atomicAdd(&wb.oor[f], (unsigned long long)oor);
}

__global__ void k_db_offsets(WinDesc wd, WinBufs wb) {
  const int f = threadIdx.x;
  if (f >= wd.n) return;
  wb.dbbeg[f] = f * wb.DBP;
  wb.dbend[f] = f * wb.DBP + (int)min(wb.dbn[f], (uint32_t)wb.DBP);
}

// D3 (+ union-find init)
__global__ void __launch_bounds__(256) k_db_gather(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const size_t o = (size_t)f * wb.DBP + j;
    const uint32_t pix = wb.dbv2[o];
    float p[3];
    db_point(F, P, (int)(pix % F.W), (int)(pix / F.W), p);
    wb.dbx[o] = make_float4(p[0], p[1], p[2], __uint_as_float(pix));
    wb.dbpar[o] = j;
    wb.dbsz[o] = 0;
  }
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < F.S; s += gridDim.x * blockDim.x)
    wb.dbbest[(size_t)f * wb.SMAX + s] = 0ull;
}

// the sorted position range of key k in frame f: [lo, hi)
__device__ __forceinline__ void db_range(const unsigned long long* K, uint32_t n, unsigned long long k, uint32_t& lo,
                                         uint32_t& hi) {
  uint32_t a = 0, b = n;
  while (a < b) { const uint32_t m = (a + b) >> 1; if (K[m] < k) a = m + 1; else b = m; }
  lo = a;
  b = n;
  while (a < b) { const uint32_t m = (a + b) >> 1; if (K[m] <= k) a = m + 1; else b = m; }
  hi = a;
}

// visit every record within eps of record j (itself included) of the same mask; fn(pos) -> false stops
template <typename Fn>
__device__ __forceinline__ void db_neighbours(const WinBufs& wb, int f, uint32_t n, uint32_t j, double e2, Fn fn) {
  const unsigned long long* K = wb.dbk2 + (size_t)f * wb.DBP;
  const float4* X = wb.dbx + (size_t)f * wb.DBP;
  const unsigned long long kj = K[j];
  const uint32_t s = (uint32_t)(kj >> 56);
  const int cx = (int)((kj >> (2 * DB_CB)) & ((1u << DB_CB) - 1)) - DB_BIAS;
  const int cy = (int)((kj >> DB_CB) & ((1u << DB_CB) - 1)) - DB_BIAS;
  const int cz = (int)(kj & ((1u << DB_CB) - 1)) - DB_BIAS;
  const float4 pj = X[j];
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        uint32_t lo, hi;
        db_range(K, n, db_cell_key(s, cx + dx, cy + dy, cz + dz), lo, hi);
        for (uint32_t q = lo; q < hi; ++q)
          if (db_d2(pj, X[q]) <= e2)
            if (!fn(q)) return;
      }
}

// D4
__global__ void __launch_bounds__(256) k_db_core(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  const double e2 = (double)P.db_eps * (double)P.db_eps;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int c = 0;
    db_neighbours(wb, f, n, j, e2, [&](uint32_t) { return ++c < P.db_min; });
    wb.dbcore[(size_t)f * wb.DBP + j] = c >= P.db_min ? 1 : 0;
  }
}

__device__ __forceinline__ uint32_t db_pix(const WinBufs& wb, int f, uint32_t q) {
  return __float_as_uint(wb.dbx[(size_t)f * wb.DBP + q].w);
}

__device__ uint32_t db_find(uint32_t* par, uint32_t x) {
  while (true) {
    const uint32_t p = __ldcg(&par[x]);
    if (p == x) return x;
    const uint32_t gp = __ldcg(&par[p]);
    if (gp != p) atomicCAS(&par[x], p, gp);
    x = p;
  }
}

// D5: roots are the records with the lowest pixel index of their component
__global__ void __launch_bounds__(256) k_db_union(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  const double e2 = (double)P.db_eps * (double)P.db_eps;
  uint32_t* par = wb.dbpar + (size_t)f * wb.DBP;
  const uint8_t* core = wb.dbcore + (size_t)f * wb.DBP;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    if (!core[j]) continue;
    db_neighbours(wb, f, n, j, e2, [&](uint32_t q) {
      if (q <= j || !core[q]) return true;   // each core pair once
      uint32_t a = j, b = q;
      while (true) {
        a = db_find(par, a);
        b = db_find(par, b);
        if (a == b) break;
        if (db_pix(wb, f, a) > db_pix(wb, f, b)) { const uint32_t t = a; a = b; b = t; }
        if (atomicCAS(&par[b], b, a) == b) break;   // the root with the higher pixel goes under the lower
      }
      return true;
    });
  }
}

// D6
__global__ void __launch_bounds__(256) k_db_label(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  const double e2 = (double)P.db_eps * (double)P.db_eps;
  uint32_t* par = wb.dbpar + (size_t)f * wb.DBP;
  const uint8_t* core = wb.dbcore + (size_t)f * wb.DBP;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    uint32_t r = U32_EMPTY;
    if (core[j]) {
      r = db_find(par, j);
    } else {
      uint32_t best_pix = U32_EMPTY;
      db_neighbours(wb, f, n, j, e2, [&](uint32_t q) {
        if (core[q]) {
          const uint32_t rq = db_find(par, q);
          const uint32_t pq = db_pix(wb, f, rq);
          if (pq < best_pix) { best_pix = pq; r = rq; }
        }
        return true;
      });
    }
    wb.dblab[(size_t)f * wb.DBP + j] = r;
    if (r != U32_EMPTY) atomicAdd(&wb.dbsz[(size_t)f * wb.DBP + r], 1u);
  }
}

// D7
__global__ void __launch_bounds__(256) k_db_best(WinDesc wd, WinBufs wb) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const size_t o = (size_t)f * wb.DBP + j;
    if (!wb.dbcore[o] || wb.dbpar[o] != j) continue;   // cluster roots only
    const uint32_t s = (uint32_t)(wb.dbk2[o] >> 56);
    const unsigned long long v = ((unsigned long long)wb.dbsz[o] << 32) | (0xFFFFFFFFu - db_pix(wb, f, j));
    atomicMax(&wb.dbbest[(size_t)f * wb.SMAX + s], v);
  }
}

// D8: the kept points into the frame tables (K1c's insertion, with K1b's key and R21 normal)
template <bool SEM>
__global__ void __launch_bounds__(256) k_db_emit(WinDesc wd, WinBufs wb, Params P, int* err) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const uint32_t n = min(wb.dbn[f], (uint32_t)wb.DBP);
  const uint32_t tmask = (uint32_t)wb.PC - 1;
  unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
  NSum* nsum = wb.nsum + (size_t)f * wb.PC;
  const float rinv = 1.0f / P.r;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const size_t o = (size_t)f * wb.DBP + j;
    const uint32_t r = wb.dblab[o];
    if (r == U32_EMPTY) continue;
    const uint32_t s = (uint32_t)(wb.dbk2[o] >> 56);
    const unsigned long long best = wb.dbbest[(size_t)f * wb.SMAX + s];
    if ((uint32_t)best != 0xFFFFFFFFu - db_pix(wb, f, r)) continue;   // not the segment's kept cluster
    const float4 x = wb.dbx[o];
    const float pc[3] = {x.x, x.y, x.z};
    uint64_t key;
    if (!point_key_fast(pc, P.r, rinv, key)) continue;   // (excluded at D1)
    const uint32_t kslot = ktab_insert(ktab, tmask, key, err);
    if (kslot == U32_EMPTY) continue;
    bool fresh = false;
    const uint32_t pslot = ptab_insert(ptab, tmask, (s << 24) | kslot, &fresh, err);
    if (pslot == U32_EMPTY) continue;
    if (SEM) {   // R21 pixel normal from the 4 neighbours' pinned world points
      const uint32_t pix = __float_as_uint(x.w);
      const int u = (int)(pix % F.W), v = (int)(pix / F.W);
      float pl[3], pr[3], pu[3], pd[3], nn[3];
      if (u >= 1 && u + 1 < F.W && v >= 1 && v + 1 < F.H && db_point(F, P, u - 1, v, pl) &&
          db_point(F, P, u + 1, v, pr) && db_point(F, P, u, v - 1, pu) && db_point(F, P, u, v + 1, pd) &&
          normal_from(F, pc, pl, pr, pu, pd, nn))
        nsum_add(&nsum[pslot], nn[0], nn[1], nn[2]);
    }
    if (fresh) {
      atomicAdd(&wb.vs[(size_t)f * wb.SMAX + s], 1u);
      const uint32_t gi = atomicAdd(&wb.npairs[f], 1u);
      if (gi < (uint32_t)wb.PMAX) wb.plist[(size_t)f * wb.PMAX + gi] = pslot;
      else raise_err(err, DERR_FRAME_PAIRS);
    }
  }
}

size_t dbscan_tmp_bytes(int n_items, int n_seg) {
  size_t b = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, b, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                           (const uint32_t*)nullptr, (uint32_t*)nullptr, n_items, n_seg,
                                           (const int*)nullptr, (const int*)nullptr, 0, 64, (cudaStream_t)0);
  return b;
}

int launch_dbscan(const WinDesc& wd, const WinBufs& wb, const Params& P, int* err, bool sem, int nsm, cudaStream_t st) {
  const int n = wd.n;
  const dim3 g(2 * nsm, n);
  cudaMemsetAsync(wb.dbn, 0, sizeof(uint32_t) * n, st);
  k_db_points<<<g, 256, 0, st>>>(wd, wb, P, err);
  k_db_offsets<<<1, 32, 0, st>>>(wd, wb);
  size_t tb = wb.dbtmp_bytes;
  cub::DeviceSegmentedRadixSort::SortPairs(wb.dbtmp, tb, wb.dbk, wb.dbk2, wb.dbv, wb.dbv2, n * wb.DBP, n, wb.dbbeg,
                                           wb.dbend, 0, 64, st);
  k_db_gather<<<g, 256, 0, st>>>(wd, wb, P);
  k_db_core<<<g, 256, 0, st>>>(wd, wb, P);
  k_db_union<<<g, 256, 0, st>>>(wd, wb, P);
  k_db_label<<<g, 256, 0, st>>>(wd, wb, P);
  k_db_best<<<g, 256, 0, st>>>(wd, wb);
  if (sem) k_db_emit<true><<<g, 256, 0, st>>>(wd, wb, P, err);
  else k_db_emit<false><<<g, 256, 0, st>>>(wd, wb, P, err);
  debug_check(st, "k_db_*", -1);
  return 10;
}

}  // namespace disc
