// k_map.cu -- stage 2 of the DISC hot path: the per-frame sequential map update
// (DESIGN.md §5).  Frame f+1's lookups depend on frame f's merges,
// so these kernels run per frame, stream-ordered.
//
//  K5  k_lookup   every unique (s, key) of the frame probes the voxel hash; each label of
//                 the key's bucket is one voxel of V_j, so c_sj += 1 (exact |V_s ∩ V_j|,
//                 P:71), warp-aggregated into a small (s, j) count table
//  K6  k_assoc    one CTA: exact fp64 threshold (R10) + pinned fp64 visual gate (R15),
//                 connected components over detections ∪ touched instances (union by
//                 min-label propagation), survivor = min id (R13), small-to-large physical
//                 label choice, pinned-order T sums and Q-gated embedding replacement
//  K7a k_apply    relabel the smaller merged sets in place (insert-if-absent root label,
//                 tombstone the old one) and insert the frame's detection voxels
//  K7b k_grow     per target: exact |V| update, grow its key-slot list
//  K7c k_fill     append new key slots to the lists
#include "disc_common.cuh"
#include "disc_launch.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace disc {

// ------------------------------------------------------------------------------------------
// voxel hash primitives
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t map_find(const MapState& M, uint64_t key) {
  uint64_t h = mix64(key) & (M.MC - 1);
  for (uint64_t probe = 0; probe < M.MC; ++probe) {
    const unsigned long long k = __ldcg(&M.slots[h].key);
    if (k == key) return (uint32_t)h;
    if (k == KEY_EMPTY) return U32_EMPTY;
    h = (h + 1) & (M.MC - 1);
  }
  return U32_EMPTY;
}

__device__ __forceinline__ uint32_t map_insert_key(const MapState& M, uint64_t key) {
  uint64_t h = mix64(key) & (M.MC - 1);
  for (uint64_t probe = 0; probe < M.MC; ++probe) {
    unsigned long long k = __ldcg(&M.slots[h].key);
    if (k == key) return (uint32_t)h;
    if (k == KEY_EMPTY) {
      k = atomicCAS(&M.slots[h].key, KEY_EMPTY, (unsigned long long)key);
      if (k == KEY_EMPTY || k == key) return (uint32_t)h;
    }
    h = (h + 1) & (M.MC - 1);
  }
  raise_err(M.err, DERR_MAP_KEYS);
  return U32_EMPTY;
}

// Insert label L into the key's label list unless present.  Linearisable because labels
// only occupy a prefix of the list (EMPTY is a suffix, never re-created) and L is only ever
// written by this routine: concurrent inserters of the same L meet at the same first EMPTY
// cell, where exactly one CAS succeeds.  Returns true iff this call inserted L.
__device__ bool label_insert(const MapState& M, uint32_t slot, uint32_t L) {
  uint32_t* labs = M.slots[slot].lab;
  int n = INLINE_LABELS;
  uint32_t* next = &M.slots[slot].ovf;
  while (true) {
    for (int i = 0; i < n; ++i) {
      const uint32_t v = __ldcg(&labs[i]);
      if (v == L) return false;
      if (v == U32_EMPTY) {
        const uint32_t old = atomicCAS(&labs[i], U32_EMPTY, L);
        if (old == U32_EMPTY) return true;
        if (old == L) return false;
      }
    }
    uint32_t nx = __ldcg(next);
    if (nx == U32_EMPTY) {
      const uint32_t c = atomicAdd(M.ovf_top, 1u);
      if (c >= M.OVFCAP) {
        raise_err(M.err, DERR_OVF_POOL);
        return false;
      }
      const uint32_t old = atomicCAS(next, U32_EMPTY, c);
      nx = (old == U32_EMPTY) ? c : old;   // a losing chunk is leaked (rare)
    }
    labs = M.ovf[nx].lab;
    n = CHUNK_LABELS;
    next = &M.ovf[nx].next;
  }
}

// Replace label L of the key by a tombstone (only the relabel of L's owner touches L).
__device__ bool label_tomb(const MapState& M, uint32_t slot, uint32_t L) {
  uint32_t* labs = M.slots[slot].lab;
  int n = INLINE_LABELS;
  uint32_t nx = __ldcg(&M.slots[slot].ovf);
  while (true) {
    for (int i = 0; i < n; ++i) {
      const uint32_t v = __ldcg(&labs[i]);
      if (v == L) {
        atomicExch(&labs[i], LAB_TOMB);
        return true;
      }
      if (v == U32_EMPTY) return false;
    }
    if (nx == U32_EMPTY) return false;
    labs = M.ovf[nx].lab;
    n = CHUNK_LABELS;
    nx = __ldcg(&M.ovf[nx].next);
  }
}

// ------------------------------------------------------------------------------------------
// K5: lookup + overlap counts
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void count_add(const FrameScratch& X, uint64_t code, uint32_t add, int* err) {
  uint32_t h = (uint32_t)mix64(code) & (uint32_t)(X.CC - 1);
  for (int probe = 0; probe < X.CC; ++probe) {
    unsigned long long k = __ldcg(&X.ctab_key[h]);
    if (k == KEY_EMPTY) {
      k = atomicCAS(&X.ctab_key[h], KEY_EMPTY, (unsigned long long)code);
      if (k == KEY_EMPTY) {
        const uint32_t t = atomicAdd(X.ntrip, 1u);
        if (t < (uint32_t)X.TCAP) {
          X.trip_s[t] = (uint32_t)(code >> 32);
          X.trip_j[t] = (uint32_t)code;
          X.ctab_idx[t] = h;   // slot of triple t
        } else {
          raise_err(err, DERR_TRIPLES);
        }
        k = code;
      }
    }
    if (k == code) {
      atomicAdd(&X.ctab_cnt[h], add);
      return;
    }
    h = (h + 1) & (uint32_t)(X.CC - 1);
  }
  raise_err(err, DERR_TRIPLES);
}

__device__ __forceinline__ void s2_lookup(int f, const WinBufs& wb, const MapState& M, const FrameScratch& X) {
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  const int lane = threadIdx.x & 31;
  unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  const int32_t* status = wb.status + (size_t)f * wb.SMAX;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < np; base += stride) {
    const uint32_t idx = base + lane;
    uint64_t code = KEY_EMPTY;   // first label's (s, j)
    uint32_t s = 0, slot = U32_EMPTY;
    if (idx < np) {
      s = wb.pinfo[fo + idx];
      ktab[wb.pfk[fo + idx]] = KEY_EMPTY;   // release the frame key-table cell
      if (status[s] == 0) {
        slot = map_find(M, wb.pkey[fo + idx]);
        if (slot != U32_EMPTY) {
          const KeySlot& ks = M.slots[slot];
          int nl = 0;
          for (int i = 0; i < INLINE_LABELS; ++i) {
            const uint32_t L = ks.lab[i];
            if (L == U32_EMPTY) break;
            if (L == LAB_TOMB) continue;
            const uint64_t c = ((uint64_t)s << 32) | M.id_of[L];
            if (nl == 0) code = c;
            else count_add(X, c, 1, M.err);
            nl++;
          }
          uint32_t nx = ks.ovf;
          while (nx != U32_EMPTY) {
            const OvfChunk& oc = M.ovf[nx];
            for (int i = 0; i < CHUNK_LABELS; ++i) {
              const uint32_t L = oc.lab[i];
              if (L == U32_EMPTY) break;
              if (L == LAB_TOMB) continue;
              const uint64_t c = ((uint64_t)s << 32) | M.id_of[L];
              if (nl == 0) code = c;
              else count_add(X, c, 1, M.err);
              nl++;
            }
            nx = oc.next;
          }
        }
      }
      wb.pms[fo + idx] = slot;
    }
    // warp aggregation of the first label's count (most keys carry one label)
    const unsigned peers = __match_any_sync(0xffffffffu, code);
    if (code != KEY_EMPTY && lane == __ffs(peers) - 1) count_add(X, code, __popc(peers), M.err);
  }
}

// ------------------------------------------------------------------------------------------
// K6: association (single CTA)
// ------------------------------------------------------------------------------------------
constexpr int K6_THREADS = 512;

__device__ __forceinline__ double dot_pin_w(const double* a, const double* b, int n) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int d = lane;
  for (; d + 96 < n; d += 128) {   // loads of four steps in flight; fma order unchanged (R15)
    const double a0 = a[d], b0 = b[d], a1 = a[d + 32], b1 = b[d + 32];
    const double a2 = a[d + 64], b2 = b[d + 64], a3 = a[d + 96], b3 = b[d + 96];
    acc = __fma_rn(a0, b0, acc);
    acc = __fma_rn(a1, b1, acc);
    acc = __fma_rn(a2, b2, acc);
    acc = __fma_rn(a3, b3, acc);
  }
  for (; d < n; d += 32) acc = __fma_rn(a[d], b[d], acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  return acc;
}

// dot_pin with every load of the lane issued before the (unchanged) fma chain
__device__ __forceinline__ double dot_pin_reg(const double* a, const double* b, int n) {
  const int lane = threadIdx.x & 31;
  double x[16], y[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int d = lane + 32 * i;
    x[i] = d < n ? a[d] : 0.0;
    y[i] = d < n ? b[d] : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (lane + 32 * i < n) acc = __fma_rn(x[i], y[i], acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  return acc;
}

struct K6Smem {   // offsets into dynamic shared memory
  size_t t_s, t_j, t_c, t_e, t_jl, lab, jnode, comp_root, comp_best, comp_tgt, has_edge, d_st, d_vs, d_tgt, d_q,
      tg_root, tg_phys, j_vc, j_ph, j_obs, j_q, total;
  __host__ __device__ K6Smem(int S, int TC) {
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t r = o; o = (o + bytes + 15) & ~(size_t)15; return r; };
    const size_t NN = (size_t)S + TC;
    t_s = take(4 * (size_t)TC); t_j = take(4 * (size_t)TC); t_c = take(4 * (size_t)TC);
    t_e = take((size_t)TC); t_jl = take(4 * (size_t)TC); lab = take(4 * NN); jnode = take(4 * (size_t)TC);
    comp_root = take(4 * NN); comp_best = take(8 * NN); comp_tgt = take(4 * NN); has_edge = take((size_t)S + 1);
    d_st = take(4 * (size_t)S + 4); d_vs = take(4 * (size_t)S + 4); d_tgt = take(4 * (size_t)S + 4);
    d_q = take(4 * (size_t)S + 4);
    tg_root = take(4 * (size_t)S + 4); tg_phys = take(4 * (size_t)S + 4);
    j_vc = take(8 * (size_t)TC); j_ph = take(4 * (size_t)TC); j_obs = take(4 * (size_t)TC); j_q = take(4 * (size_t)TC);
    total = o;
  }
};

// DISC_K6PROF: phase timestamps of the association kernel (profiling aid)
__device__ unsigned long long g_k6prof[16];
__device__ unsigned long long g_s2prof[8];   // DISC_S2PROF phase sums
#define K6_PROBE(i)                                                                          \
  do {                                                                                       \
    if (threadIdx.x == 0) {                                                                  \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      atomicAdd(&g_k6prof[(i) + 1], t_ - g_k6prof[0]);                                        \
      g_k6prof[0] = t_;                                                                      \
    }                                                                                        \
  } while (0)

__device__ __forceinline__ void s2_assoc(int f, const FrameDesc& F, const WinBufs& wb, const MapState& M,
                                         const FrameScratch& X, const Params& P, int sem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TC = X.TCAP;
  const int S = F.S;
  const K6Smem L6(S, TC);
  uint32_t* t_s = (uint32_t*)(smem_raw + L6.t_s);          // triple s
  uint32_t* t_j = (uint32_t*)(smem_raw + L6.t_j);          // triple j (instance id)
  uint32_t* t_c = (uint32_t*)(smem_raw + L6.t_c);          // c_sj
  uint8_t* t_e = (uint8_t*)(smem_raw + L6.t_e);            // edge flag
  int32_t* t_jl = (int32_t*)(smem_raw + L6.t_jl);          // local instance index
  int32_t* lab = (int32_t*)(smem_raw + L6.lab);            // [S + nJ] component label
  uint32_t* jnode = (uint32_t*)(smem_raw + L6.jnode);      // local index -> id
  uint32_t* comp_root = (uint32_t*)(smem_raw + L6.comp_root);
  unsigned long long* comp_best = (unsigned long long*)(smem_raw + L6.comp_best);
  int32_t* comp_tgt = (int32_t*)(smem_raw + L6.comp_tgt);
  uint8_t* has_edge = (uint8_t*)(smem_raw + L6.has_edge);
  int32_t* d_st = (int32_t*)(smem_raw + L6.d_st);     // per-detection status (staged from global)
  uint32_t* d_vs = (uint32_t*)(smem_raw + L6.d_vs);   // |V_s|
  int32_t* d_tgt = (int32_t*)(smem_raw + L6.d_tgt);   // target index (written back at the end)
  float* d_q = (float*)(smem_raw + L6.d_q);           // Q_s
  uint32_t* tg_root = (uint32_t*)(smem_raw + L6.tg_root);   // per target: survivor id
  uint32_t* tg_phys = (uint32_t*)(smem_raw + L6.tg_phys);   // per target: physical label
  int64_t* j_vc = (int64_t*)(smem_raw + L6.j_vc);           // per local instance: |V_j|
  uint32_t* j_ph = (uint32_t*)(smem_raw + L6.j_ph);         //   physical label
  int32_t* j_obs = (int32_t*)(smem_raw + L6.j_obs);         //   obs count
  float* j_q = (float*)(smem_raw + L6.j_q);                 //   Q
  __shared__ uint32_t n_tr, n_j, n_tgt, n_seg, ncomp_s;
  __shared__ uint32_t mcnt_s[256], dcnt_s[256], moff_s[256], doff_s[256];
  __shared__ int64_t tg_vb[256];
  __shared__ int changed;
  __shared__ unsigned long long rel_s, merged_s, edges_s;
  __shared__ uint32_t gen;

  const size_t fo = (size_t)f * wb.SMAX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  if (tid == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_k6prof[0] = t_;
  }
  if (tid == 0) {
    n_tr = min(*X.ntrip, (uint32_t)TC);
    if (*X.ntrip > (uint32_t)TC) raise_err(M.err, DERR_TRIPLES);
    n_j = 0; n_tgt = 0; n_seg = 0; rel_s = 0; merged_s = 0; edges_s = 0;
    gen = (uint32_t)(++M.counters[3]);
    *X.nstage = 0;
    *X.nrel = 0;
  }
  for (int i = tid; i < S + TC; i += blockDim.x) {
    lab[i] = i;
    comp_root[i] = U32_EMPTY;
    comp_best[i] = 0;
    comp_tgt[i] = -1;
  }
  for (int i = tid; i < S; i += blockDim.x) {
    has_edge[i] = 0;
    d_tgt[i] = -1;
    d_st[i] = wb.status[fo + i];
    d_vs[i] = wb.vs[fo + i];
    d_q[i] = wb.qf[(fo + i) * 6 + 4];
    X.det_id[i] = -1;
    X.tgt_stage[i] = 0;
  }
  __syncthreads();
  K6_PROBE(0);
  const uint32_t ntr = n_tr;
  // ---- triples: load and release the count table ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    const uint32_t h = X.ctab_idx[t];
    t_s[t] = X.trip_s[t];
    t_j[t] = X.trip_j[t];
    t_c[t] = X.ctab_cnt[h];
    X.ctab_cnt[h] = 0;
    X.ctab_key[h] = KEY_EMPTY;
  }
  __syncthreads();
  K6_PROBE(1);
  // ---- O10 edges: exact fp64 geometric test (R10) + pinned fp64 visual gate (R15) ----
  const double* trk = wb.trk + fo * P.Dt;
  for (uint32_t t = warp; t < ntr; t += nwarp) {
    const uint32_t s = t_s[t], j = t_j[t], c = t_c[t];
    const int64_t vs = d_vs[s], vj = M.vcount[j];
    const int64_t mn = vs < vj ? vs : vj;
    bool e = c >= 1 && (double)c >= (double)P.tau_geo * (double)mn;
    if (e && P.Dt > 0) {
      const double* Tj = M.T + (size_t)j * P.Dt;
      const double TT = M.TT[j];
      const double dt = dot_pin_reg(trk + (size_t)s * P.Dt, Tj, P.Dt);
      double cosv = -2.0;
      if (wb.tok[fo + s] && TT > 0.0) cosv = __ddiv_rn(dt, __dsqrt_rn(TT));
      e = cosv >= (double)P.tau_vis;
    }
    if (lane == 0) t_e[t] = e ? 1 : 0;
  }
  __syncthreads();
  K6_PROBE(2);
  // ---- distinct instances among the edges -> local node S + l (generation stamps) ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    if (!t_e[t]) continue;
    has_edge[t_s[t]] = 1;
    const uint32_t j = t_j[t];
    if (atomicExch(&M.stamp[j], gen) != gen) {
      const uint32_t l = atomicAdd(&n_j, 1u);
      M.local[j] = (int32_t)l;
      jnode[l] = j;
    }
  }
  __syncthreads();
  K6_PROBE(3);
  for (uint32_t t = tid; t < ntr; t += blockDim.x) t_jl[t] = t_e[t] ? M.local[t_j[t]] : -1;
  for (int l = tid; l < (int)n_j; l += blockDim.x) {   // one parallel round of attribute loads
    const uint32_t j = jnode[l];
    j_vc[l] = M.vcount[j];
    j_ph[l] = M.phys_of[j];
    j_obs[l] = M.obs[j];
    j_q[l] = M.q[j];
  }
  __syncthreads();
  K6_PROBE(4);
  const int nJ = (int)n_j;
  const int NN = S + nJ;
  // ---- O11 components: min-label propagation with pointer jumping ----
  while (true) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (uint32_t t = tid; t < ntr; t += blockDim.x) {
      if (!t_e[t]) continue;
      const int a = (int)t_s[t], b = S + t_jl[t];
      const int la = lab[a], lb = lab[b];
      if (la != lb) {
        const int m = la < lb ? la : lb;
        atomicMin(&lab[a], m);
        atomicMin(&lab[b], m);
        atomicMin(&lab[la], m);
        atomicMin(&lab[lb], m);
        changed = 1;
      }
    }
    __syncthreads();
    for (int x = tid; x < NN; x += blockDim.x) {
      int l = lab[x];
      while (lab[l] != l) l = lab[l];
      lab[x] = l;
    }
    __syncthreads();
    if (!changed) break;
    __syncthreads();
  }
  // ---- per component: root = min id (R13), physical owner = max |V| (ties: min id) ----
  for (int l = tid; l < nJ; l += blockDim.x) {
    const int Lb = lab[S + l];
    const uint32_t j = jnode[l];
    atomicMin(&comp_root[Lb], j);
    const unsigned long long key = ((unsigned long long)(uint64_t)j_vc[l] << 32) | (0x7FFFFFFFu - j);
    atomicMax(&comp_best[Lb], key);
  }
  __syncthreads();
  K6_PROBE(5);
  for (int x = tid; x < NN; x += blockDim.x) {
    if (lab[x] == x && comp_root[x] != U32_EMPTY) {
      const int t = (int)atomicAdd(&n_tgt, 1u);
      comp_tgt[x] = t;
      const uint32_t owner = 0x7FFFFFFFu - (uint32_t)(comp_best[x] & 0xFFFFFFFFull);
      tg_root[t] = comp_root[x];
      tg_phys[t] = M.phys_of[owner];
      tg_vb[t] = (int64_t)(comp_best[x] >> 32);   // |V| of the physical owner
    }
  }
  __syncthreads();
  K6_PROBE(6);
  // ---- detections: component members, isolated kept ones -> new ids ascending s (R13) ----
  if (tid == 0) {
    ncomp_s = n_tgt;
    int64_t nid = M.counters[0];
    int64_t created = 0;
    for (int s = 0; s < S; ++s) {
      if (d_st[s] != 0) continue;
      if (has_edge[s]) {
        const int t = comp_tgt[lab[s]];
        d_tgt[s] = t;
        X.det_id[s] = tg_root[t];
      } else {
        if (nid >= M.IMAX) {
          raise_err(M.err, DERR_INSTANCES);
          break;
        }
        const int t = (int)n_tgt++;
        d_tgt[s] = t;
        X.det_id[s] = nid;
        tg_root[t] = (uint32_t)nid;
        tg_phys[t] = (uint32_t)nid;
        nid++;
        created++;
      }
    }
    M.counters[0] = nid;
    M.counters[1] += created;
    X.rep[f].created = created;
  }
  __syncthreads();
  K6_PROBE(7);
  // ---- O12 work lists for K7a (one CTA per target): member ids ascending, detections
  // ascending; relabel segments for the smaller sets; report sums ----
  const int ncomp = (int)ncomp_s;
  const int ntg = (int)n_tgt;
  for (int t = tid; t <= S; t += blockDim.x) { mcnt_s[t] = 0; dcnt_s[t] = 0; }
  __syncthreads();
  for (int l = tid; l < nJ; l += blockDim.x) atomicAdd(&mcnt_s[comp_tgt[lab[S + l]]], 1u);
  if (tid == 0) {
    for (int s2 = 0; s2 < S; ++s2)
      if (d_tgt[s2] >= 0) dcnt_s[d_tgt[s2]]++;
    uint32_t mo = 0, dof = 0;
    for (int t = 0; t < ntg; ++t) {
      moff_s[t] = mo; mo += mcnt_s[t];
      doff_s[t] = dof; dof += dcnt_s[t];
      dcnt_s[t] = 0;
    }
    for (int s2 = 0; s2 < S; ++s2) {
      const int t = d_tgt[s2];
      if (t >= 0) X.tg_dets[doff_s[t] + dcnt_s[t]++] = (uint32_t)s2;
    }
  }
  __syncthreads();
  for (int l = tid; l < nJ; l += blockDim.x) {
    const int t = comp_tgt[lab[S + l]];
    const uint32_t j = jnode[l];
    uint32_t rank = 0;
    for (int l2 = 0; l2 < nJ; ++l2)
      if (l2 != l && comp_tgt[lab[S + l2]] == t && jnode[l2] < j) rank++;
    X.tg_mem[moff_s[t] + rank] = j;
    const uint32_t pm = j_ph[l];
    if (pm != tg_phys[t]) {   // the smaller sets: relabel into the survivor's physical label
      const uint32_t sg = atomicAdd(&n_seg, 1u);
      if (sg < (uint32_t)TC) {
        X.seg_phys[sg] = pm;
        X.seg_tgt[sg] = t;
        X.seg_base[sg] = M.lst_off[pm];
        X.seg_off[sg] = M.lst_len[pm];
      } else {
        raise_err(M.err, DERR_TRIPLES);
      }
    }
    if (j != tg_root[t]) {
      atomicAdd(&rel_s, (unsigned long long)j_vc[l]);
      atomicAdd(&merged_s, 1ull);
    }
  }
  for (int t = tid; t < ntg; t += blockDim.x) {
    X.tgt_root[t] = tg_root[t];
    X.tgt_phys[t] = tg_phys[t];
    X.tg_kind[t] = t < ncomp ? 0 : 1;
    X.tg_vbase[t] = t < ncomp ? tg_vb[t] : 0;
    X.tg_moff[t] = moff_s[t];
    X.tg_mcnt[t] = mcnt_s[t];
    X.tg_doff[t] = doff_s[t];
    X.tg_dcnt[t] = dcnt_s[t];
  }
  for (int s2 = tid; s2 < S; s2 += blockDim.x) X.det_target[s2] = d_tgt[s2];
  __syncthreads();
  K6_PROBE(8);
  // ---- debug copies of the triples, edge count ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    X.trip_c[t] = t_c[t];
    X.trip_edge[t] = t_e[t];
    if (t_e[t]) atomicAdd(&edges_s, 1ull);
  }
  __syncthreads();
  K6_PROBE(9);
  if (tid == 0) {
    const uint32_t ns = min(n_seg, (uint32_t)TC);
    uint32_t acc = 0;
    for (uint32_t g = 0; g < ns; ++g) {
      const uint32_t len = X.seg_off[g];
      X.seg_off[g] = acc;
      acc += len;
    }
    X.seg_off[ns] = acc;
    *X.nseg = (int)ns;
    *X.nrel = acc;
    *X.ntgt = (int)n_tgt;
    disc_frame_report& R = X.rep[f];
    int kept = 0, da = 0, dc = 0, dasp = 0, dnd = 0, dnf = 0;
    int64_t U = 0;
    for (int s = 0; s < S; ++s) {
      switch (d_st[s]) {
        case 0: kept++; U += d_vs[s]; break;
        case 1: da++; break;
        case 2: dc++; break;
        case 3: dasp++; break;
        case 4: dnd++; break;
        default: dnf++; break;
      }
    }
    R.kept = kept; R.drop_area = da; R.drop_conf = dc; R.drop_aspect = dasp;
    R.drop_nodepth = dnd; R.drop_nofeat = dnf;
    R.key_out_of_range = (int64_t)wb.oor[f];
    R.unique_pairs = U;
    R.edges = (int64_t)edges_s;
    M.counters[4] += U;
    M.counters[7] += (int64_t)edges_s;
    M.counters[6] += (int64_t)acc;
    R.merged_away = (int64_t)merged_s;
    R.relabeled = (int64_t)rel_s;
    M.counters[1] -= (int64_t)merged_s;
    R.live_instances = M.counters[1];
    *X.live_before = M.counters[2];
    *X.ntrip_last = ntr;
    *X.ntrip = 0;
  }
}

// ------------------------------------------------------------------------------------------
// K7a: apply.  Blocks [0, ntgt) first execute one O12 target each (instance-table update of a
// merged component / creation of a new instance); then every block joins the grid-stride loop
// of detection inserts and small-to-large relabels.
// ------------------------------------------------------------------------------------------
constexpr int K7_T = 256;

__device__ void apply_target(int t, int f, const FrameDesc& F, const WinBufs& wb, const MapState& M,
                             const FrameScratch& X, const Params& P, int sem) {
  __shared__ float q_s[K7_T];
  __shared__ int32_t ab_s[6];
  __shared__ int32_t obs_s;
  __shared__ int src_s;            // -1 keep, i < mcnt member i, mcnt + k detection k
  const int tid = threadIdx.x, lane = tid & 31;
  const size_t fo = (size_t)f * wb.SMAX;
  const double* trk = wb.trk + fo * P.Dt;
  const int kind = X.tg_kind[t];
  const uint32_t root = X.tgt_root[t], L = X.tgt_phys[t];
  const uint32_t moff = X.tg_moff[t], mcnt = X.tg_mcnt[t], doff = X.tg_doff[t], dcnt = X.tg_dcnt[t];
  const uint32_t* mem = X.tg_mem + moff;
  const uint32_t* dets = X.tg_dets + doff;
  if (kind == 1) {   // new instance from its single detection (O12 last paragraph)
    const uint32_t s = dets[0], id = root;
    const float qs = wb.qf[(fo + s) * 6 + 4];
    if (tid == 0) {
      M.alive[id] = 1;
      M.phys_of[id] = id;
      M.id_of[id] = id;
      M.vcount[id] = 0;
      M.obs[id] = 1;
      M.last_seen[id] = F.frame_id;
      for (int k = 0; k < 6; ++k) M.aabb[(size_t)id * 6 + k] = wb.daabb[(fo + s) * 6 + k];
      M.q[id] = qs;
      M.lst_len[id] = 0;
      M.lst_cap[id] = 0;
    }
    for (int d = tid; d < P.Dt; d += blockDim.x) M.T[(size_t)id * P.Dt + d] = trk[(size_t)s * P.Dt + d];
    const bool has_e = sem && qs >= 0.f;
    for (int d = tid; d < P.Df; d += blockDim.x) M.E[(size_t)id * P.Df + d] = has_e ? wb.emb[(fo + s) * P.Df + d] : 0.f;
    if (P.Dt > 0 && tid < 32) {
      const double tt = dot_pin_reg(trk + (size_t)s * P.Dt, trk + (size_t)s * P.Dt, P.Dt);
      if (lane == 0) M.TT[id] = tt;
    }
    return;
  }
  // merged component: root = mem[0] (min id), J = mem[1..], Sd = dets (ascending)
  if (tid == 0) {
    obs_s = 0;
    for (int k = 0; k < 3; ++k) { ab_s[k] = INT32_MAX; ab_s[3 + k] = INT32_MIN; }
  }
  __syncthreads();
  int myobs = 0;
  for (uint32_t i = tid; i < mcnt + dcnt; i += blockDim.x) {
    const int32_t* ab;
    if (i < mcnt) {
      const uint32_t m = mem[i];
      myobs += M.obs[m];
      ab = M.aabb + (size_t)m * 6;
      if (i < K7_T) q_s[i] = M.q[m];
    } else {
      const uint32_t s = dets[i - mcnt];
      myobs += 1;
      ab = wb.daabb + (fo + s) * 6;
      if (i < K7_T) q_s[i] = wb.qf[(fo + s) * 6 + 4];
    }
    for (int k = 0; k < 3; ++k) {
      atomicMin(&ab_s[k], ab[k]);
      atomicMax(&ab_s[3 + k], ab[3 + k]);
    }
  }
  if (myobs) atomicAdd(&obs_s, myobs);
  // T_root <- ((T_root + T_j1) + T_j2 ...) + t_s1 ...   elementwise fp64, exactly this order
  double* Tr = M.T + (size_t)root * P.Dt;
  for (int d = tid; d < P.Dt; d += blockDim.x) {
    double acc = Tr[d];
    for (uint32_t i = 1; i < mcnt; ++i) acc = __dadd_rn(acc, M.T[(size_t)mem[i] * P.Dt + d]);
    for (uint32_t k = 0; k < dcnt; ++k) acc = __dadd_rn(acc, trk[(size_t)dets[k] * P.Dt + d]);
    Tr[d] = acc;
  }
  __syncthreads();
  // (e, Q): root's, then J ascending, then Sd ascending, replace iff Q_cand > Q (strict)
  if (tid == 0) {
    float qcur = q_s[0];
    int src = -1;
    for (uint32_t i = 1; i < mcnt + dcnt; ++i) {
      const float qi = i < K7_T ? q_s[i] : (i < mcnt ? M.q[mem[i]] : wb.qf[(fo + dets[i - mcnt]) * 6 + 4]);
      if (qi > qcur) { qcur = qi; src = (int)i; }
    }
    src_s = src;
    q_s[0] = qcur;
  }
  if (P.Dt > 0 && tid < 32) {
    const double tt = dot_pin_reg(Tr, Tr, P.Dt);
    if (lane == 0) M.TT[root] = tt;
  }
  __syncthreads();
  const int src = src_s;
  if (src >= 0) {
    const float* e = (uint32_t)src < mcnt ? M.E + (size_t)mem[src] * P.Df : wb.emb + (fo + dets[src - mcnt]) * P.Df;
    for (int d = tid; d < P.Df; d += blockDim.x) M.E[(size_t)root * P.Df + d] = e[d];
  }
  // members: key lists of physical labels other than the survivor's were captured by K6 as
  // relabel segments; reset them, kill J
  for (uint32_t i = tid; i < mcnt; i += blockDim.x) {
    const uint32_t m = mem[i];
    const uint32_t pm = M.phys_of[m];
    if (pm != L) {
      M.lst_len[pm] = 0;
      M.lst_cap[pm] = 0;
    }
  }
  __syncthreads();
  for (uint32_t i = 1 + tid; i < mcnt; i += blockDim.x) {
    const uint32_t m = mem[i];
    M.alive[m] = 0;
    M.phys_of[m] = U32_EMPTY;
  }
  if (tid == 0) {
    M.obs[root] = obs_s;
    M.last_seen[root] = F.frame_id;
    for (int k = 0; k < 6; ++k) M.aabb[(size_t)root * 6 + k] = ab_s[k];
    M.q[root] = q_s[0];
    M.vcount[root] = X.tg_vbase[t];
    M.phys_of[root] = L;
    M.id_of[L] = root;
  }
}

__device__ __forceinline__ void s2_apply(int f, const FrameDesc& F, const WinBufs& wb, const MapState& M,
                                         const FrameScratch& X, const Params& P, int sem) {
  for (int t = blockIdx.x; t < *X.ntgt; t += gridDim.x) {
    apply_target(t, f, F, wb, M, X, P, sem);
    __syncthreads();
  }
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const uint32_t nrel = *X.nrel;
  const uint32_t total = np + nrel;
  const size_t fo = (size_t)f * wb.PMAX;
  const int nseg = *X.nseg;
  const int lane = threadIdx.x & 31;
  __shared__ int delta_s;
  if (threadIdx.x == 0) delta_s = 0;
  __syncthreads();
  int delta = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < total; base += stride) {
    const uint32_t it = base + lane;
    int tnew = -1;
    uint32_t snew = 0;
    if (it < np) {
      const uint32_t s = wb.pinfo[fo + it];
      const int t = X.det_target[s];
      if (t >= 0) {
        const uint32_t L = X.tgt_phys[t];
        uint32_t slot = wb.pms[fo + it];
        if (slot == U32_EMPTY) slot = map_insert_key(M, wb.pkey[fo + it]);
        if (slot != U32_EMPTY && label_insert(M, slot, L)) { tnew = t; snew = slot; delta++; }
      }
    } else if (it < total) {
      const uint32_t r = it - np;
      int lo = 0, hi = nseg - 1;   // last segment with seg_off <= r
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (X.seg_off[mid] <= r) lo = mid;
        else hi = mid - 1;
      }
      const int t = X.seg_tgt[lo];
      const uint32_t L = X.tgt_phys[t];
      const uint32_t slot = M.arena[X.seg_base[lo] + (r - X.seg_off[lo])];
      if (label_insert(M, slot, L)) { tnew = t; snew = slot; delta++; }
      if (label_tomb(M, slot, X.seg_phys[lo])) delta--;
    }
    // warp-aggregated staging of the new (target, slot) entries
    const unsigned peers = __match_any_sync(0xffffffffu, tnew);
    if (tnew >= 0 && lane == __ffs(peers) - 1) atomicAdd(&X.tgt_stage[tnew], (uint32_t)__popc(peers));
    const unsigned b = __ballot_sync(0xffffffffu, tnew >= 0);
    if (b) {
      uint32_t sb = 0;
      if (lane == 0) sb = atomicAdd(X.nstage, (uint32_t)__popc(b));
      sb = __shfl_sync(0xffffffffu, sb, 0);
      if (tnew >= 0) {
        const uint32_t i = sb + __popc(b & ((1u << lane) - 1u));
        if (i < X.STCAP) {
          X.stage_slot[i] = snew;
          X.stage_tgt[i] = (uint32_t)tnew;
        } else {
          raise_err(M.err, DERR_STAGE);
        }
      }
    }
  }
  if (delta) atomicAdd(&delta_s, delta);
  __syncthreads();
  if (threadIdx.x == 0 && delta_s) atomicAdd((unsigned long long*)&M.counters[2], (unsigned long long)(int64_t)delta_s);
}

// K7b: per target — |V| update and list growth
__device__ __forceinline__ void s2_grow(int f, const MapState& M, const FrameScratch& X) {
  const int ntgt = *X.ntgt;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    disc_frame_report& R = X.rep[f];
    R.live_memberships = M.counters[2];
    R.new_memberships = M.counters[2] - *X.live_before;
  }
  for (int t = blockIdx.x; t < ntgt; t += gridDim.x) {
  __syncthreads();
  const uint32_t L = X.tgt_phys[t];
  const uint32_t root = X.tgt_root[t];
  const uint32_t add = X.tgt_stage[t];
  __shared__ unsigned long long newoff;
  __shared__ uint32_t oldlen, grow;
  if (threadIdx.x == 0) {
    M.vcount[root] += add;
    oldlen = M.lst_len[L];
    const uint32_t need = oldlen + add;
    grow = 0;
    if (need > M.lst_cap[L]) {
      const uint32_t nc = max(max(2 * M.lst_cap[L], need), 64u);
      const unsigned long long off = atomicAdd(M.arena_top, (unsigned long long)nc);
      if (off + nc > M.ARENA) {
        raise_err(M.err, DERR_ARENA);
      } else {
        newoff = off;
        grow = 1;
        M.lst_cap[L] = nc;
      }
    }
    X.tgt_base[t] = oldlen;
    X.tgt_fill[t] = 0;
  }
  __syncthreads();
  if (grow) {
    const unsigned long long src = M.lst_off[L];
    for (uint32_t i = threadIdx.x; i < oldlen; i += blockDim.x) M.arena[newoff + i] = M.arena[src + i];
    __syncthreads();
    if (threadIdx.x == 0) M.lst_off[L] = newoff;
  }
  if (threadIdx.x == 0) {
    M.lst_len[L] = oldlen + add;
    atomicAdd((unsigned long long*)&M.counters[5], (unsigned long long)add);
  }
  }
}

// K7c: fill the appended list cells (warp-aggregated positions)
__device__ __forceinline__ void s2_fill(const MapState& M, const FrameScratch& X) {
  const uint32_t n = min(*X.nstage, X.STCAP);
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const uint32_t i = base + lane;
    const int t = i < n ? (int)X.stage_tgt[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, t);
    const int leader = __ffs(peers) - 1;
    uint32_t pb = 0;
    if (t >= 0 && lane == leader) pb = atomicAdd(&X.tgt_fill[t], (uint32_t)__popc(peers));
    pb = __shfl_sync(0xffffffffu, pb, leader);
    if (t >= 0) {
      const uint32_t L = X.tgt_phys[t];
      const uint32_t pos = X.tgt_base[t] + pb + __popc(peers & ((1u << lane) - 1u));
      M.arena[M.lst_off[L] + pos] = X.stage_slot[i];
    }
  }
}

size_t k6_smem_bytes(int S, int TC) { return K6Smem(S, TC).total; }

void k6_prof_dump() {
  if (getenv("DISC_S2PROF")) {
    unsigned long long g[8];
    cudaMemcpyFromSymbol(g, g_s2prof, sizeof(g));
    fprintf(stderr, "s2 phase ns: lookup %llu assoc %llu apply %llu grow %llu fill %llu\n", g[0], g[1], g[2], g[3], g[4]);
  }
  unsigned long long h[16];
  cudaMemcpyFromSymbol(h, g_k6prof, sizeof(h));
  fprintf(stderr, "k6 phase ns (cumulative):");
  for (int i = 1; i < 12; ++i) fprintf(stderr, " %d:%llu", i - 1, h[i]);
  fprintf(stderr, "\n");
}

// Grid-wide barrier of the persistent stage-2 kernel (all CTAs co-resident: the grid is sized to
// the SMs K1 leaves free, one CTA per SM).  Monotonic counter, zeroed by K0 for the window.
__device__ __forceinline__ void grid_sync(uint32_t* bar, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// Stage 2 of a window: the frames' map updates in order, five grid-synchronised phases per frame
// (K5 lookup, K6 association on CTA 0, K7a apply, K7b grow, K7c fill) in one persistent launch.
__global__ void __launch_bounds__(K6_THREADS, 1) k_stage2(WinDesc wd, WinBufs wb, MapState M, FrameScratch X,
                                                        Params P, int sem, int prof) {
  const uint32_t G = gridDim.x;
  uint32_t ep = 0;
  unsigned long long t_prev = 0;
  auto probe = [&](int i) {   // DISC_S2PROF: phase durations on CTA 0 (profiling aid)
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      if (i >= 0) atomicAdd(&g_s2prof[i], t_ - t_prev);
      t_prev = t_;
    }
  };
  probe(-1);
  for (int f = 0; f < wd.n; ++f) {
    const FrameDesc& F = wd.f[f];
    s2_lookup(f, wb, M, X);
    grid_sync(wb.s2bar, G * ++ep);
    probe(0);
    if (blockIdx.x == 0) s2_assoc(f, F, wb, M, X, P, sem);
    grid_sync(wb.s2bar, G * ++ep);
    probe(1);
    s2_apply(f, F, wb, M, X, P, sem);
    grid_sync(wb.s2bar, G * ++ep);
    probe(2);
    s2_grow(f, M, X);
    grid_sync(wb.s2bar, G * ++ep);
    probe(3);
    s2_fill(M, X);
    grid_sync(wb.s2bar, G * ++ep);
    probe(4);
  }
}

int launch_stage2(const WinDesc& wd, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P,
                  bool sem, int nsm, int nres, cudaStream_t st) {
  const size_t sm6 = k6_smem_bytes(wb.SMAX, X.TCAP);
  static size_t set_for = 0;
  if (set_for != sm6) {
    cudaFuncSetAttribute(k_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
    set_for = sm6;
  }
  const int grid = nres > 0 ? nres : std::min(16, nsm);
  static const int prof = getenv("DISC_S2PROF") ? 1 : 0;
  k_stage2<<<grid, K6_THREADS, sm6, st>>>(wd, wb, M, X, P, sem ? 1 : 0, prof);
  debug_check(st, "k_stage2", -1);
  return 1;
}

}  // namespace disc
