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

// As map_insert_key, with the home slot tried by a CAS first (no read when it is free);
// *created = this call claimed the slot (its label cells are all EMPTY).
__device__ __forceinline__ uint32_t map_insert_key_c(const MapState& M, uint64_t key, bool* created) {
  uint64_t h = mix64(key) & (M.MC - 1);
  unsigned long long k = atomicCAS(&M.slots[h].key, KEY_EMPTY, (unsigned long long)key);
  if (k == KEY_EMPTY) { *created = true; return (uint32_t)h; }
  if (k == key) return (uint32_t)h;
  for (uint64_t probe = 1; probe < M.MC; ++probe) {
    h = (h + 1) & (M.MC - 1);
    k = __ldcg(&M.slots[h].key);
    if (k == key) return (uint32_t)h;
    if (k == KEY_EMPTY) {
      k = atomicCAS(&M.slots[h].key, KEY_EMPTY, (unsigned long long)key);
      if (k == KEY_EMPTY) { *created = true; return (uint32_t)h; }
      if (k == key) return (uint32_t)h;
    }
  }
  raise_err(M.err, DERR_MAP_KEYS);
  return U32_EMPTY;
}

struct SlotV {   // a KeySlot read as two 16-byte L2 loads (key and inline labels together)
  unsigned long long key;
  uint32_t lab[INLINE_LABELS];
  uint32_t ovf;
};
__device__ __forceinline__ SlotV slot_load(const MapState& M, uint32_t h) {
  const uint4* p = reinterpret_cast<const uint4*>(M.slots + h);
  const uint4 a = __ldcg(p), b = __ldcg(p + 1);
  SlotV v;
  v.key = (unsigned long long)a.x | ((unsigned long long)a.y << 32);
  v.lab[0] = a.z; v.lab[1] = a.w; v.lab[2] = b.x; v.lab[3] = b.y; v.lab[4] = b.z;
  v.ovf = b.w;
  return v;
}

// Insert label L into the key's label list unless present.  Linearisable because labels
// only occupy a prefix of the list (EMPTY is a suffix, never re-created) and L is only ever
// written by this routine: concurrent inserters of the same L meet at the same first EMPTY
// cell, where exactly one CAS succeeds.  Returns true iff this call inserted L.
__device__ bool label_insert(const MapState& M, uint32_t slot, uint32_t L) {
  for (;;) {   // inline labels: one 32-byte read, then a CAS on the first EMPTY cell
    const SlotV v = slot_load(M, slot);
    int e = -1;
#pragma unroll
    for (int i = 0; i < INLINE_LABELS; ++i) {
      if (e >= 0) continue;
      if (v.lab[i] == L) return false;
      if (v.lab[i] == U32_EMPTY) e = i;
    }
    if (e < 0) break;   // inline cells full: overflow chunks
    const uint32_t old = atomicCAS(&M.slots[slot].lab[e], U32_EMPTY, L);
    if (old == U32_EMPTY) return true;
    if (old == L) return false;
  }
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
// A frame's (s, j) count table: table 0 (FrameScratch's ctab_* / ntrip / trip_s / trip_j) or table
// 1 (the *2 fields; speculative counting alternates them between consecutive frames)
struct CTab {
  unsigned long long* key;
  uint32_t *cnt, *idx, *ntrip, *ts, *tj;
  int32_t CC, TCAP;
};
__device__ __forceinline__ CTab ctab(const FrameScratch& X, int p) {
  CTab C;
  C.key = p ? X.ctab_key2 : X.ctab_key;
  C.cnt = p ? X.ctab_cnt2 : X.ctab_cnt;
  C.idx = p ? X.ctab_idx2 : X.ctab_idx;
  C.ntrip = p ? X.ntrip2 : X.ntrip;
  C.ts = p ? X.trip_s2 : X.trip_s;
  C.tj = p ? X.trip_j2 : X.trip_j;
  C.CC = X.CC;
  C.TCAP = X.TCAP;
  return C;
}

__device__ __forceinline__ void count_add(const CTab& X, uint64_t code, uint32_t add, int* err) {
  uint32_t h = (uint32_t)mix64(code) & (uint32_t)(X.CC - 1);
  for (int probe = 0; probe < X.CC; ++probe) {
    unsigned long long k = __ldcg(&X.key[h]);
    if (k == KEY_EMPTY) {
      k = atomicCAS(&X.key[h], KEY_EMPTY, (unsigned long long)code);
      if (k == KEY_EMPTY) {
        const uint32_t t = atomicAdd(X.ntrip, 1u);
        if (t < (uint32_t)X.TCAP) {
          X.ts[t] = (uint32_t)(code >> 32);
          X.tj[t] = (uint32_t)code;
          X.idx[t] = h;   // slot of triple t
        } else {
          raise_err(err, DERR_TRIPLES);
        }
        k = code;
      }
    }
    if (k == code) {
      atomicAdd(&X.cnt[h], add);
      return;
    }
    h = (h + 1) & (uint32_t)(X.CC - 1);
  }
  raise_err(err, DERR_TRIPLES);
}

// LK_Q pairs per lane, their hash probes in lockstep, so each lane keeps LK_Q independent
// memory chains in flight (the lookup is a latency chain: attributes -> slot -> labels ->
// count table).
#ifndef LK_AGG2
#define LK_AGG2 1   // warp-aggregate the second label too (0: round-1 behaviour, per-lane shared atomics)
#endif
#ifndef LK_REV
#define LK_REV 1
#endif
#ifndef LK_Q
#define LK_Q 1   // unique (s, key) pairs per lane in flight.  The persistent kernel shares one register
                 // allocation: LK_Q 3 spilled 664 B per thread across all phases, 2 316 B, 1 72 B (H
                 // bench r02: M1 14.3 k / 15.1 k / 16.5 k frames/s)
#endif
// DISC_S2PROF: lookup sub-phases on the first CTA of the lookup (init, loop, flush; loop steps 3..8),
// [0..9] the per-frame lookup phase, [10..19] the speculative counting
__device__ unsigned long long g_lkprof[20];
__device__ __forceinline__ void lk_probe(int i, unsigned long long& tp, int b0) {
  if (blockIdx.x == (unsigned)b0 && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    if (i >= 0) atomicAdd(&g_lkprof[i + (b0 ? 10 : 0)], t_ - tp);
    tp = t_;
  }
}
constexpr int LK_CT = 2048;   // per-CTA (s, j) count table slots (in the dynamic shared memory)

// spec: the pair's slot index was found by s2_spec during the previous frame's association (pms,
// U32_EMPTY = key absent then): keys never move in the open-addressing table, so the probe starts
// at that slot and matches at once; only keys absent then (new keys) probe from their home slot
//
// b0 > 0: run on CTAs b0.. only.  tag != 0: the speculative counting of frame f during the
// previous frame's association -- a kept pair whose key is absent gets the key's slot created (no
// labels: counts nothing; K7 of this frame fills it anyway), and every kept pair is chained onto its
// slot (M.slh[slot] = tag << 32 | pair, wb.pnext) for the previous frame's K7 to find the pairs whose
// counts its label changes correct.
__device__ __forceinline__ void s2_lookup(int f, const WinBufs& wb, const MapState& M, const FrameScratch& X,
                                          const CTab& C, bool spec = false, int b0 = 0, uint32_t tag = 0) {
  const uint32_t np = min(__ldcg(&wb.npairs[f]), (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  const int lane = threadIdx.x & 31;
  // the association's shared memory is free during this phase: a CTA table of (s, j) counts
  // (flushed to the frame's count table at the end)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* ck = (unsigned long long*)smem_raw;                 // [LK_CT] codes
  uint32_t* cc = (uint32_t*)(ck + LK_CT);                                 // [LK_CT] counts
  const int32_t* stf = wb.status + (size_t)f * wb.SMAX;                   // the frame's statuses
  unsigned long long tp = 0;
  lk_probe(-1, tp, b0);
  for (int i = threadIdx.x; i < LK_CT; i += blockDim.x) { ck[i] = KEY_EMPTY; cc[i] = 0; }
  __syncthreads();
  lk_probe(0, tp, b0);
  auto cta_add = [&](uint64_t code, uint32_t add) {   // CTA table, else straight to the frame's
    uint32_t h = (uint32_t)mix64(code) & (LK_CT - 1);
    for (int probe = 0; probe < 64; ++probe) {
      unsigned long long k = ck[h];
      if (k == KEY_EMPTY) {
        k = atomicCAS(&ck[h], KEY_EMPTY, (unsigned long long)code);
        if (k == KEY_EMPTY) k = code;
      }
      if (k == code) {
        atomicAdd(&cc[h], add);
        return;
      }
      h = (h + 1) & (LK_CT - 1);
    }
    count_add(C, code, add, M.err);
  };
  const uint32_t nb = gridDim.x - b0;
  const uint32_t stride = LK_Q * nb * blockDim.x;
  const uint32_t hmask = (uint32_t)(M.MC - 1);
  const uint32_t gthreads = nb * blockDim.x;
  // pair q of a lane: base + q * (grid threads), so every CTA gets an equal share
  // (speculative counting: CTA b takes share G-1-b, so CTAs 1.., which evaluate the visual gate
  // first, get the last shares -- one pair per lane where the first shares have two)
  const uint32_t cb = b0 > 0 && LK_REV ? gridDim.x - 1 - blockIdx.x : blockIdx.x - b0;
  for (uint32_t base = cb * blockDim.x + (threadIdx.x & ~31u); base < np; base += stride) {
    uint32_t idx[LK_Q], s[LK_Q], slot[LK_Q], h[LK_Q];
    unsigned long long key[LK_Q];
    bool act[LK_Q];
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) {
      idx[q] = base + q * gthreads + lane;
      s[q] = 0; slot[q] = U32_EMPTY; key[q] = KEY_EMPTY; act[q] = false;
      if (idx[q] < np) {
        s[q] = wb.pinfo[fo + idx[q]];
        key[q] = wb.pkey[fo + idx[q]];
        DBOUND(s[q] < (uint32_t)wb.SMAX, M.err);
      }
    }
    lk_probe(7, tp, b0);   // pair records loaded
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) {
      act[q] = idx[q] < np && stf[s[q]] == 0;   // (a few L1 lines: no staging round trip)
      h[q] = (uint32_t)mix64(key[q]) & hmask;
      if (spec && idx[q] < np) {
        const uint32_t ps = wb.pms[fo + idx[q]];
        if (ps != U32_EMPTY) h[q] = ps;
      }
    }
    bool kept[LK_Q];
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) kept[q] = act[q];
    SlotV sv[LK_Q];
    auto any_act = [&]() {
      bool a = false;
#pragma unroll
      for (int q = 0; q < LK_Q; ++q) a = a || act[q];
      return a;
    };
    for (uint32_t probe = 0; any_act() && probe <= hmask; ++probe) {
#pragma unroll
      for (int q = 0; q < LK_Q; ++q)
        if (act[q]) sv[q] = slot_load(M, h[q]);
#pragma unroll
      for (int q = 0; q < LK_Q; ++q) {
        if (!act[q]) continue;
        if (sv[q].key == key[q]) { slot[q] = h[q]; act[q] = false; }
        else if (sv[q].key == KEY_EMPTY) act[q] = false;
        else h[q] = (h[q] + 1) & hmask;
      }
    }
    lk_probe(3, tp, b0);   // status + probes done
    if (tag) {   // (speculative counting) absent keys created, every kept pair chained onto its slot
#pragma unroll
      for (int q = 0; q < LK_Q; ++q) {
        if (kept[q] && slot[q] == U32_EMPTY) {
          bool created = false;
          slot[q] = map_insert_key_c(M, key[q], &created);
          DBOUND(slot[q] == U32_EMPTY || slot[q] < M.MC, M.err);
          sv[q].lab[0] = sv[q].lab[1] = U32_EMPTY;   // (a slot created now has no labels)
          sv[q].ovf = U32_EMPTY;
#pragma unroll
          for (int i = 2; i < INLINE_LABELS; ++i) sv[q].lab[i] = U32_EMPTY;
        }
      }
      unsigned long long old[LK_Q];
#pragma unroll
      for (int q = 0; q < LK_Q; ++q)
        if (kept[q] && slot[q] != U32_EMPTY)
          old[q] = atomicExch(&M.slh[slot[q]], ((unsigned long long)tag << 32) | idx[q]);
#pragma unroll
      for (int q = 0; q < LK_Q; ++q)
        if (kept[q] && slot[q] != U32_EMPTY)
          wb.pnext[fo + idx[q]] = (uint32_t)(old[q] >> 32) == tag ? (uint32_t)old[q] : U32_EMPTY;
      lk_probe(8, tp, b0);   // slot chains (their exchanges' round trip)
    }
    // each pair's first two live labels (s, j) are counted warp-aggregated (a frame's keys mostly carry
    // one or two labels, and a warp's pairs mostly the same ones: per-lane shared atomics on one hot
    // counter serialise); further labels (rare) directly
    uint64_t first[LK_Q], second[LK_Q];
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) { first[q] = KEY_EMPTY; second[q] = KEY_EMPTY; }
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) {
      if (idx[q] < np) {
        wb.pms[fo + idx[q]] = slot[q];
        // labels only ever gain entries, except the tombstones of merged-away sets, never the
        // survivor's: a label present now is present when K7 would insert it
        wb.plab[fo + idx[q]] = slot[q] == U32_EMPTY ? make_uint2(U32_EMPTY, U32_EMPTY)
                                                    : make_uint2(sv[q].lab[0], sv[q].lab[1]);
      }
      if (slot[q] == U32_EMPTY) continue;
      uint32_t id[INLINE_LABELS];
      bool ok[INLINE_LABELS];
      bool open = true;   // no EMPTY met yet (labels occupy a prefix)
#pragma unroll
      for (int i = 0; i < INLINE_LABELS; ++i) {
        const uint32_t L = sv[q].lab[i];
        if (L == U32_EMPTY) open = false;
        ok[i] = open && L != LAB_TOMB;
        id[i] = ok[i] ? L : 0u;   // counted by physical label (one-to-one with the live ids here)
      }
      int nl = 0;
#pragma unroll
      for (int i = 0; i < INLINE_LABELS; ++i) {
        if (!ok[i]) continue;
        const uint64_t c = ((uint64_t)s[q] << 32) | id[i];
        if (nl == 0) first[q] = c;
        else if (LK_AGG2 && nl == 1) second[q] = c;
        else cta_add(c, 1);
        nl++;
      }
      if (open) {   // overflow chunks (more than INLINE_LABELS labels on this key)
        uint32_t nx = sv[q].ovf;
        while (nx != U32_EMPTY) {
          const OvfChunk& oc = M.ovf[nx];
          for (int i = 0; i < CHUNK_LABELS; ++i) {
            const uint32_t L = __ldcg(&oc.lab[i]);
            if (L == U32_EMPTY) break;
            if (L == LAB_TOMB) continue;
            const uint64_t c = ((uint64_t)s[q] << 32) | L;
            if (nl == 0) first[q] = c;
            else if (LK_AGG2 && nl == 1) second[q] = c;
            else cta_add(c, 1);
            nl++;
          }
          nx = __ldcg(&oc.next);
        }
      }
    }
    lk_probe(4, tp, b0);   // labels walked, records stored
#pragma unroll
    for (int q = 0; q < LK_Q; ++q) {   // warp aggregation of the first (and second) label's count
      const unsigned peers = __match_any_sync(0xffffffffu, first[q]);
      if (first[q] != KEY_EMPTY && lane == __ffs(peers) - 1) cta_add(first[q], __popc(peers));
      if (LK_AGG2) {
        const unsigned p2 = __match_any_sync(0xffffffffu, second[q]);
        if (second[q] != KEY_EMPTY && lane == __ffs(p2) - 1) cta_add(second[q], __popc(p2));
      }
    }
    lk_probe(5, tp, b0);   // aggregated
  }
  lk_probe(-1, tp, b0);
  __syncthreads();
  lk_probe(6, tp, b0);   // barrier: the CTA's slowest warp
  lk_probe(1, tp, b0);
  for (int i = threadIdx.x; i < LK_CT; i += blockDim.x)   // flush the CTA's counts
    if (cc[i]) count_add(C, ck[i], cc[i], M.err);
  __syncthreads();
  lk_probe(2, tp, b0);
}

// ------------------------------------------------------------------------------------------
// K6: association (single CTA)
// ------------------------------------------------------------------------------------------
#ifndef K6_T
#define K6_T 512
#endif
constexpr int K6_THREADS = K6_T;

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

struct K6Smem {   // offsets into dynamic shared memory
  size_t t_s, t_j, t_c, t_e, t_jl, lab, jnode, comp_root, comp_best, comp_tgt, has_edge, d_st, d_vs, d_tgt, d_q,
      tg_root, tg_phys, j_vc, j_ph, j_obs, j_q, j_lo, j_ll, j_lc, total;
  __host__ __device__ K6Smem(int S, int TC) {
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t r = o; o = (o + bytes + 15) & ~(size_t)15; return r; };
    const size_t NN = (size_t)S + TC;
    t_s = take((size_t)TC); t_j = take(4 * (size_t)TC); t_c = take(4 * (size_t)TC);
    t_e = take((size_t)TC); t_jl = take(4 * (size_t)TC); lab = take(4 * NN); jnode = take(4 * (size_t)TC);
    comp_root = take(4 * NN); comp_best = take(8 * NN); comp_tgt = take(4 * NN); has_edge = take((size_t)S + 1);
    d_st = take(4 * (size_t)S + 4); d_vs = take(4 * (size_t)S + 4); d_tgt = take(4 * (size_t)S + 4);
    d_q = take(4 * (size_t)S + 4);
    tg_root = take(4 * (size_t)S + 4); tg_phys = take(4 * (size_t)S + 4);
    j_vc = take(4 * (size_t)TC); j_ph = take(4 * (size_t)TC); j_obs = take(4 * (size_t)TC); j_q = take(4 * (size_t)TC);
    j_lo = take(4 * (size_t)TC); j_ll = take(4 * (size_t)TC); j_lc = take(4 * (size_t)TC);   // list of the phys label
    total = o;
  }
};

// DISC_K6PROF: phase timestamps of the association kernel (profiling aid)
__device__ unsigned long long g_k6prof[16];
__device__ unsigned long long g_s2prof[8];   // DISC_S2PROF phase sums
__device__ unsigned long long g_s2cta[8];
__device__ unsigned long long g_s2items[4];
__device__ unsigned long long g_tgprof[4];   // DISC_S2PROF: target-update warp time sum / max, count
__device__ unsigned long long g_approf[8];
__device__ unsigned long long g_s2place[4];   // k_stage2 CTA placement: launches, CTAs, CTAs on SMs >= the grid size
__device__ unsigned long long g_tghist[24];   // DISC_S2PROF: target time sum / count / max by candidates (new, <=2, <=4, <=8, <=16, <=32, more)   // DISC_S2PROF: K7 sub-steps, per-frame maxima [0..3], summed [4..7]
#define K6_PROBE(i)                                                                          \
  do {                                                                                       \
    if (threadIdx.x == 0) {                                                                  \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      atomicAdd(&g_k6prof[(i) + 1], t_ - g_k6prof[0]);                                        \
      g_k6prof[0] = t_;                                                                      \
    }                                                                                        \
  } while (0)

// fresh: the CTA's static shared counters are not known to be zero (first frame of a launch); later
// frames find them zeroed by the previous frame's association, and skip one barrier
__device__ __forceinline__ void s2_assoc(int f, const FrameDesc& F, const WinBufs& wb, const MapState& M,
                                         const FrameScratch& X, const CTab& C, const Params& P, int sem,
                                         bool fresh = true, bool dbg = true) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // Layout: the shared-memory tables hold up to X.TCS (s, j) triples; a denser frame (hierarchical
  // SAM-"everything" masks overlapping many instances, BASELINE configs[4]) runs the same steps on
  // the same layout in a global-memory scratch sized for X.TCAP triples (block-scope atomics and
  // __syncthreads order it exactly as in shared memory).  Only a frame past X.TCAP fails (loudly).
  const uint32_t ntr_all = __ldcg(C.ntrip);
  const uint32_t ntr = min(ntr_all, (uint32_t)X.TCAP);
  const bool gmode = ntr > (uint32_t)X.TCS;
  const int TC = gmode ? X.TCAP : X.TCS;
  unsigned char* const k6b = gmode ? X.k6g : smem_raw;
  const int S = F.S;
  const K6Smem L6(S, TC);
  uint8_t* t_s = (uint8_t*)(k6b + L6.t_s);            // triple s (S <= 255)
  uint32_t* t_j = (uint32_t*)(k6b + L6.t_j);          // triple j (instance id)
  uint32_t* t_c = (uint32_t*)(k6b + L6.t_c);          // c_sj
  uint8_t* t_e = (uint8_t*)(k6b + L6.t_e);            // edge flag
  int32_t* t_jl = (int32_t*)(k6b + L6.t_jl);          // local instance index
  int32_t* lab = (int32_t*)(k6b + L6.lab);            // [S + nJ] component label
  uint32_t* jnode = (uint32_t*)(k6b + L6.jnode);      // local index -> id
  uint32_t* comp_root = (uint32_t*)(k6b + L6.comp_root);
  unsigned long long* comp_best = (unsigned long long*)(k6b + L6.comp_best);
  int32_t* comp_tgt = (int32_t*)(k6b + L6.comp_tgt);
  uint8_t* has_edge = (uint8_t*)(k6b + L6.has_edge);
  int32_t* d_st = (int32_t*)(k6b + L6.d_st);     // per-detection status (staged from global)
  uint32_t* d_vs = (uint32_t*)(k6b + L6.d_vs);   // |V_s|
  int32_t* d_tgt = (int32_t*)(k6b + L6.d_tgt);   // target index (written back at the end)
  float* d_q = (float*)(k6b + L6.d_q);           // Q_s
  uint32_t* tg_root = (uint32_t*)(k6b + L6.tg_root);   // per target: survivor id
  uint32_t* tg_phys = (uint32_t*)(k6b + L6.tg_phys);   // per target: physical label
  uint32_t* j_vc = (uint32_t*)(k6b + L6.j_vc);         // per local instance: |V_j|
  uint32_t* j_lo = (uint32_t*)(k6b + L6.j_lo);         //   key list of its physical label: offset,
  uint32_t* j_ll = (uint32_t*)(k6b + L6.j_ll);         //   length,
  uint32_t* j_lc = (uint32_t*)(k6b + L6.j_lc);         //   capacity
  uint32_t* j_ph = (uint32_t*)(k6b + L6.j_ph);         //   physical label
  int32_t* j_obs = (int32_t*)(k6b + L6.j_obs);         //   obs count
  float* j_q = (float*)(k6b + L6.j_q);                 //   Q
  __shared__ uint32_t n_j, n_tgt, n_seg, ncomp_s, n_cand;
  __shared__ uint32_t mcnt_s[256], dcnt_s[256], moff_s[256], doff_s[256];
  __shared__ int64_t tg_vb[256];
  __shared__ int32_t tg_own[256];   // component target -> local index of its physical owner
  __shared__ int changed;
  __shared__ uint32_t wcnt_s[K6_THREADS / 32], wcnt2_s[K6_THREADS / 32], rc_s[8], nrel_s, bound_s[256];
  __shared__ unsigned long long rel_s, merged_s, edges_s;
  __shared__ uint32_t gen;
  __shared__ int64_t cnt_s[3];

  const size_t fo = (size_t)f * wb.SMAX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  if (tid == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_k6prof[0] = t_;
  }
  if (tid == 0) {
    if (ntr_all > (uint32_t)X.TCAP) raise_err(M.err, DERR_TRIPLES);
    if (fresh) { n_j = 0; n_tgt = 0; n_seg = 0; rel_s = 0; merged_s = 0; edges_s = 0; n_cand = 0; }
    // the map counters this step reads, all in one round trip (only this thread writes 0, 1, 3,
    // 4, 6, 7; counter 2 is K7's)
    const int64_t c0 = M.counters[0], c1 = M.counters[1], c2 = M.counters[2], c3 = M.counters[3];
    cnt_s[0] = c0; cnt_s[1] = c1; cnt_s[2] = c2;
    gen = (uint32_t)(c3 + 1);
    M.counters[3] = c3 + 1;
    *X.nrel = 0;
    *X.work = 0;
  }
  for (int i = tid; i < S + (int)ntr; i += blockDim.x) {   // nodes: detections + (<= ntr) instances
    lab[i] = i;
    comp_root[i] = U32_EMPTY;
    comp_best[i] = 0;
    comp_tgt[i] = -1;
  }
  if (fresh) __syncthreads();   // the zeroed counters above (n_cand before the triples' atomics)
  for (int i = tid; i < S; i += blockDim.x) {   // (loads in flight with the triples' below)
    has_edge[i] = 0;
    d_tgt[i] = -1;
    d_st[i] = wb.status[fo + i];
    d_vs[i] = wb.vs[fo + i];
    d_q[i] = wb.qf[(fo + i) * 6 + 4];
    X.det_id[i] = -1;
    X.tgt_stage[i] = 0;
  }
  K6_PROBE(0);
  // ---- triples (count table released) + O10 exact fp64 geometric test (R10), thread per
  // triple; candidates for the visual gate are compacted ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    const uint32_t h = C.idx[t];
    // the lookup counted by physical label: its live id (after the previous frame's update every
    // label in the map is a live instance's physical label)
    const uint32_t s = C.ts[t], j = __ldcg(&M.id_of[C.tj[t]]);
    const uint32_t c = C.cnt[h];
    const int64_t vj = M.vcount[j];
    C.cnt[h] = 0;
    C.key[h] = KEY_EMPTY;
    t_s[t] = (uint8_t)s;
    t_j[t] = j;
    t_c[t] = c;
    const int64_t vs = wb.vs[fo + s];
    const int64_t mn = vs < vj ? vs : vj;
    const bool e = c >= 1 && (double)c >= (double)P.tau_geo * (double)mn;
    t_e[t] = e ? 1 : 0;
    if (e && P.Dt > 0) t_jl[atomicAdd(&n_cand, 1u)] = (int32_t)t;   // t_jl: candidate list for now
  }
  __syncthreads();
  K6_PROBE(1);
  // ---- pinned fp64 visual gate (R15): computed for every triple by CTAs 1.. (s2_gate) while
  // this CTA ran the steps above; a single-CTA grid gates its candidates itself ----
  const double* trk = wb.trk + fo * P.Dt;
  if (P.Dt > 0 && gridDim.x > 1) {
    if (tid == 0) {
      uint32_t v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(X.gate_done) : "memory");
      } while (v < ntr);
    }
    __syncthreads();
    for (uint32_t t = tid; t < ntr; t += blockDim.x)
      if (t_e[t] && !__ldcg(&X.trip_gate[t])) t_e[t] = 0;
    if (tid == 0) *X.gate_done = 0;   // every gate of this frame is in
  } else if (P.Dt > 0) {
    const uint32_t nc = n_cand;
    for (uint32_t k = warp; k < nc; k += nwarp) {
      const uint32_t t = (uint32_t)t_jl[k];
      const uint32_t s = t_s[t], j = t_j[t];
      const double* Tj = M.T + (size_t)j * P.Dt;
      const double TT = M.TT[j];
      const uint8_t tok = wb.tok[fo + s];
      const double dt = dot_pin_reg(trk + (size_t)s * P.Dt, Tj, P.Dt);
      double cosv = -2.0;
      if (tok && TT > 0.0) cosv = __ddiv_rn(dt, __dsqrt_rn(TT));
      if (lane == 0 && !(cosv >= (double)P.tau_vis)) t_e[t] = 0;
    }
  }
  __syncthreads();
  K6_PROBE(2);
  // ---- distinct instances among the edges -> local node S + l (generation stamps) ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    if (!t_e[t]) continue;
    has_edge[t_s[t]] = 1;
    const uint32_t j = t_j[t];
    if (atomicExch(&M.stamp[j], gen) != gen) {   // first sight: local index + attributes
      const uint32_t l = atomicAdd(&n_j, 1u);
      M.local[j] = (int32_t)l;
      jnode[l] = j;
      j_vc[l] = (uint32_t)M.vcount[j];
      j_ph[l] = M.phys_of[j];
      j_obs[l] = M.obs[j];
      j_q[l] = M.q[j];
    }
  }
  __syncthreads();
  K6_PROBE(3);
  for (uint32_t t = tid; t < ntr; t += blockDim.x) t_jl[t] = t_e[t] ? __ldcg(&M.local[t_j[t]]) : -1;
  for (int l = tid; l < (int)n_j; l += blockDim.x) {   // the key list of each instance's physical label
    const uint32_t pm = j_ph[l];
    j_lo[l] = (uint32_t)M.lst_off[pm];
    j_ll[l] = M.lst_len[pm];
    j_lc[l] = M.lst_cap[pm];
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
      tg_root[t] = comp_root[x];
      tg_vb[t] = (int64_t)(comp_best[x] >> 32);   // |V| of the physical owner
    }
  }
  __syncthreads();
  for (int l = tid; l < nJ; l += blockDim.x) {   // the physical owner's local index -> its label
    const int Lb = lab[S + l];
    if (jnode[l] == 0x7FFFFFFFu - (uint32_t)(comp_best[Lb] & 0xFFFFFFFFull)) {
      tg_phys[comp_tgt[Lb]] = j_ph[l];
      tg_own[comp_tgt[Lb]] = l;
    }
  }
  __syncthreads();
  K6_PROBE(6);
  // ---- detections: component members, isolated kept ones -> new ids ascending s (R13); the
  // rank of an isolated detection among them is a block-wide exclusive count ----
  {
    const int s = tid;
    const bool kept = s < S && d_st[s] == 0;
    const bool iso = kept && !has_edge[s];
    const unsigned b = __ballot_sync(0xffffffffu, iso);
    if (lane == 0) wcnt_s[warp] = __popc(b);
    __syncthreads();
    int before = __popc(b & ((1u << lane) - 1u)), created = 0;
    for (int w2 = 0; w2 < nwarp; ++w2) {
      if (w2 < warp) before += wcnt_s[w2];
      created += wcnt_s[w2];
    }
    const int ncomp = (int)n_tgt;
    const int64_t nid0 = cnt_s[0];
    if (kept && has_edge[s]) {
      const int t = comp_tgt[lab[s]];
      d_tgt[s] = t;
      X.det_id[s] = tg_root[t];
    } else if (iso) {
      const int64_t nid = nid0 + before;
      if (nid < M.IMAX) {
        const int t = ncomp + before;
        d_tgt[s] = t;
        X.det_id[s] = nid;
        tg_root[t] = (uint32_t)nid;
        tg_phys[t] = (uint32_t)nid;
      } else {
        raise_err(M.err, DERR_INSTANCES);
      }
    }
    __syncthreads();
    if (tid == 0) {
      ncomp_s = ncomp;
      n_tgt = ncomp + created;
      M.counters[0] = nid0 + created;
      cnt_s[1] += created;
      X.rep[f].created = created;
    }
  }
  __syncthreads();
  K6_PROBE(7);
  // ---- O12 work lists for K7a (one CTA per target): member ids ascending, detections
  // ascending; relabel segments for the smaller sets; report sums ----
  const int ncomp = (int)ncomp_s;
  const int ntg = (int)n_tgt;
  for (int t = tid; t <= S; t += blockDim.x) { mcnt_s[t] = 0; dcnt_s[t] = 0; bound_s[t] = 0; }
  __syncthreads();
  for (int l = tid; l < nJ; l += blockDim.x) atomicAdd(&mcnt_s[comp_tgt[lab[S + l]]], 1u);
  for (int s2 = tid; s2 < S; s2 += blockDim.x)
    if (d_tgt[s2] >= 0) {
      atomicAdd(&dcnt_s[d_tgt[s2]], 1u);
      atomicAdd(&bound_s[d_tgt[s2]], d_vs[s2]);   // at most |V_s| new entries per detection
    }
  __syncthreads();
  {   // exclusive offsets over the targets (ntg <= S <= 255 < blockDim): warp scans + warp totals
    const int t = tid;
    uint32_t mc = t < ntg ? mcnt_s[t] : 0u, dc = t < ntg ? dcnt_s[t] : 0u;
    uint32_t mi = mc, di = dc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, mi, o), b2 = __shfl_up_sync(0xffffffffu, di, o);
      if (lane >= o) { mi += a; di += b2; }
    }
    if (lane == 31) { wcnt_s[warp] = mi; wcnt2_s[warp] = di; }
    __syncthreads();
    uint32_t mb = 0, db = 0;
    for (int w2 = 0; w2 < warp; ++w2) { mb += wcnt_s[w2]; db += wcnt2_s[w2]; }
    if (t < ntg) { moff_s[t] = mb + mi - mc; doff_s[t] = db + di - dc; }
  }
  __syncthreads();
  int32_t* tl_s = (int32_t*)comp_root;   // (comp_root is dead after the targets were formed)
  for (int l = tid; l < nJ; l += blockDim.x) tl_s[l] = comp_tgt[lab[S + l]];   // member -> target
  for (int s2 = tid; s2 < S; s2 += blockDim.x) {   // detections of each target, ascending s
    const int t = d_tgt[s2];
    if (t < 0) continue;
    uint32_t rank = 0;
#pragma unroll 8
    for (int s3 = 0; s3 < s2; ++s3) rank += d_tgt[s3] == t;
    X.tg_dets[doff_s[t] + rank] = (uint32_t)s2;
    if (mcnt_s[t] + rank < 32) X.tg_cand[t * 32 + mcnt_s[t] + rank] = (uint32_t)s2;
  }
  __syncthreads();
  for (int l = tid; l < nJ; l += blockDim.x) {
    const int t = tl_s[l];
    const uint32_t j = jnode[l];
    uint32_t rank = 0;
#pragma unroll 8
    for (int l2 = 0; l2 < nJ; ++l2) rank += (tl_s[l2] == t) & (jnode[l2] < j);   // ids are distinct
    X.tg_mem[moff_s[t] + rank] = j;
    if (rank < 32) X.tg_cand[t * 32 + rank] = j;
    const uint32_t pm = j_ph[l];
    if (pm != tg_phys[t]) {   // the smaller sets: relabel into the survivor's physical label
      const uint32_t sg = atomicAdd(&n_seg, 1u);
      if (sg < (uint32_t)TC) {
        X.seg_phys[sg] = pm;
        X.seg_tgt[sg] = t;
        X.seg_base[sg] = j_lo[l];
        const uint32_t len = j_ll[l];
        t_jl[sg] = (int32_t)len;   // segment length (t_jl is free after the components)
        atomicAdd(&bound_s[t], len);
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
  // ---- triple ids (refinement, debug export), debug copies (a window's last frame: the only one the
  // export reads), edge count; nothing below reads them before the next barrier ----
  for (uint32_t t = tid; t < ntr; t += blockDim.x) {
    C.tj[t] = t_j[t];   // (the gate CTAs are done with the labels; k_refine reads table 0's)
    if (dbg) {
      X.trip_sd[t] = t_s[t];
      X.trip_jd[t] = t_j[t];
      X.trip_c[t] = t_c[t];
      X.trip_edge[t] = t_e[t];
    }
    if (t_e[t]) atomicAdd(&edges_s, 1ull);
  }
  K6_PROBE(9);
  // relabel segment offsets: block-wide exclusive scan of the lengths (chunk per thread)
  const uint32_t ns = min(n_seg, (uint32_t)TC);
  if (ns == 0) {   // (no merge this frame: nothing to scan)
    if (tid == 0) {
      X.seg_off[0] = 0;
      nrel_s = 0;
    }
  } else {
    const uint32_t per = (ns + blockDim.x - 1) / blockDim.x;
    const uint32_t g0 = min(ns, tid * per), g1 = min(ns, g0 + per);
    uint32_t sum = 0;
    for (uint32_t g = g0; g < g1; ++g) sum += (uint32_t)t_jl[g];
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (lane == 31) wcnt_s[warp] = inc;
    __syncthreads();
    uint32_t base = inc - sum, all = 0;
    for (int w2 = 0; w2 < nwarp; ++w2) {
      if (w2 < warp) base += wcnt_s[w2];
      all += wcnt_s[w2];
    }
    for (uint32_t g = g0; g < g1; ++g) {
      X.seg_off[g] = base;
      base += (uint32_t)t_jl[g];
    }
    if (tid == 0) {
      X.seg_off[ns] = all;
      nrel_s = all;
    }
  }
  __syncthreads();
  K6_PROBE(10);
  // list capacity: each target's key list is sized for its worst-case growth this frame (one
  // entry per frame pair of its detections and per relabel item of its segments), moving it to
  // a larger arena region when needed, so K7 appends in place
  for (int t = tid; t < (int)n_tgt; t += blockDim.x) {
    const uint32_t L = tg_phys[t];
    const bool fresh = t >= (int)ncomp_s;   // new instance: empty list
    const int lo = fresh ? 0 : tg_own[t];
    const uint32_t oldlen = fresh ? 0u : j_ll[lo], cap = fresh ? 0u : j_lc[lo];
    const unsigned long long off = fresh ? 0ull : j_lo[lo];
    const uint32_t need = oldlen + bound_s[t];
    unsigned long long newoff = off, movesrc = ~0ull;
    if (need > cap) {
      const uint32_t nc = max(max(2 * cap, need), 64u);
      const unsigned long long o = atomicAdd(M.arena_top, (unsigned long long)nc);
      if (o + nc > M.ARENA) {
        raise_err(M.err, DERR_ARENA);
      } else {
        if (oldlen) movesrc = off;
        newoff = o;
        M.lst_off[L] = o;
        M.lst_cap[L] = nc;
      }
    }
    X.tgt_base[t] = oldlen;
    X.tg_newoff[t] = newoff;
    X.tg_movesrc[t] = movesrc;
    bound_s[t] = movesrc != ~0ull ? oldlen : 0u;   // entries K7 copies to the new region
  }
  __syncthreads();
  {   // prefix offsets of the copy items over the targets (n_tgt <= S < blockDim)
    const int t = tid;
    const uint32_t c = t < (int)n_tgt ? bound_s[t] : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (lane == 31) wcnt2_s[warp] = inc;
    __syncthreads();
    uint32_t base = 0, all = 0;
    for (int w2 = 0; w2 < nwarp; ++w2) {
      if (w2 < warp) base += wcnt2_s[w2];
      all += wcnt2_s[w2];
    }
    if (t < (int)n_tgt) X.tg_mvoff[t] = base + inc - c;
    if (t == 0) X.tg_mvoff[n_tgt] = all;
  }
  __syncthreads();
  K6_PROBE(11);
  // report counts (O13): statuses and U over the detections
  if (tid < 8) rc_s[tid] = 0;
  __syncthreads();
  for (int s2 = tid; s2 < S; s2 += blockDim.x) {
    const int st = d_st[s2];
    atomicAdd(&rc_s[st < 5 ? st : 5], 1u);
    if (st == 0) atomicAdd(&rc_s[6], d_vs[s2]);
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t acc = nrel_s;
    *X.nseg = (int)ns;
    *X.nrel = acc;
    *X.ntgt = (int)n_tgt;
    disc_frame_report& R = X.rep[f];
    const int64_t U = rc_s[6];
    R.kept = rc_s[0]; R.drop_area = rc_s[1]; R.drop_conf = rc_s[2]; R.drop_aspect = rc_s[3];
    R.drop_nodepth = rc_s[4]; R.drop_nofeat = rc_s[5];
    R.key_out_of_range = (int64_t)wb.oor[f];
    R.unique_pairs = U;
    R.edges = (int64_t)edges_s;
    atomicAdd((unsigned long long*)&M.counters[4], (unsigned long long)U);
    atomicAdd((unsigned long long*)&M.counters[7], (unsigned long long)edges_s);
    atomicAdd((unsigned long long*)&M.counters[6], (unsigned long long)acc);
    R.merged_away = (int64_t)merged_s;
    R.relabeled = (int64_t)rel_s;
    R.refine_rounds = 0;   // (k_refine adds to these when refine_active)
    R.refine_merged = 0;
    const int64_t live = cnt_s[1] - (int64_t)merged_s;
    M.counters[1] = live;
    R.live_instances = live;
    *X.live_before = cnt_s[2];
    *X.ntrip_last = ntr;
    *C.ntrip = 0;
  }
  __syncthreads();
  if (tid == 0) { n_j = 0; n_tgt = 0; n_seg = 0; rel_s = 0; merged_s = 0; edges_s = 0; n_cand = 0; }   // next frame
  K6_PROBE(12);
}

// ------------------------------------------------------------------------------------------
// K7a: apply.  Blocks [0, ntgt) first execute one O12 target each (instance-table update of a
// merged component / creation of a new instance); then every block joins the grid-stride loop
// of detection inserts and small-to-large relabels.
// ------------------------------------------------------------------------------------------
// One O12 target per warp (a few dozen per frame), so every target runs at once and the warps
// without one start the inserts immediately.
__device__ void apply_target_warp_general(int t, int f, const FrameDesc& F, const WinBufs& wb,
                                                  const MapState& M, const FrameScratch& X, const Params& P, int sem) {
  const int lane = threadIdx.x & 31;
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
    if (lane == 0) {
      M.alive[id] = 1;
      M.phys_of[id] = id;
      M.id_of[id] = id;
      M.vcount[id] = 0;
      M.obs[id] = 1;
      M.last_seen[id] = F.frame_id;
      M.q[id] = qs;
      M.lst_len[id] = 0;
    }
    if (lane < 6) M.aabb[(size_t)id * 6 + lane] = wb.daabb[(fo + s) * 6 + lane];
    for (int d = lane; d < P.Dt; d += 32) M.T[(size_t)id * P.Dt + d] = trk[(size_t)s * P.Dt + d];
    const bool has_e = sem && qs >= 0.f;
    const float4* es = (const float4*)(wb.emb + (fo + s) * P.Df);
    float4* ed = (float4*)(M.E + (size_t)id * P.Df);
    for (int d4 = lane; d4 < P.Df / 4; d4 += 32) ed[d4] = has_e ? es[d4] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (P.Dt > 0) {
      const double tt = dot_pin_reg(trk + (size_t)s * P.Dt, trk + (size_t)s * P.Dt, P.Dt);
      if (lane == 0) M.TT[id] = tt;
    }
    return;
  }
  // merged component: root = mem[0] (min id), J = mem[1..], Sd = dets (ascending)
  const uint32_t n = mcnt + dcnt;
  int obs = 0;
  int32_t ab[6] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN};
  float qbest = -INFINITY;   // max Q over candidates 1..n-1, first index attaining it
  int ibest = -1;
  float q0 = 0.f;
  for (uint32_t i0 = 0; i0 < n; i0 += 32) {
    const uint32_t i = i0 + lane;
    float qi = -INFINITY;
    if (i < n) {
      const int32_t* a;
      if (i < mcnt) {
        const uint32_t m = mem[i];
        obs += M.obs[m];
        a = M.aabb + (size_t)m * 6;
        qi = M.q[m];
      } else {
        const uint32_t s = dets[i - mcnt];
        obs += 1;
        a = wb.daabb + (fo + s) * 6;
        qi = wb.qf[(fo + s) * 6 + 4];
      }
      for (int k = 0; k < 3; ++k) { ab[k] = min(ab[k], a[k]); ab[3 + k] = max(ab[3 + k], a[3 + k]); }
    }
    if (i0 == 0) q0 = __shfl_sync(0xffffffffu, qi, 0);
    const bool cand = i >= 1 && i < n;
    float qm = cand ? qi : -INFINITY;
#pragma unroll
    for (int o = 16; o; o >>= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
    const unsigned hit = __ballot_sync(0xffffffffu, cand && qi == qm);
    if (qm > qbest && hit) { qbest = qm; ibest = (int)i0 + __ffs(hit) - 1; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    obs += __shfl_xor_sync(0xffffffffu, obs, o);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      ab[k] = min(ab[k], __shfl_xor_sync(0xffffffffu, ab[k], o));
      ab[3 + k] = max(ab[3 + k], __shfl_xor_sync(0xffffffffu, ab[3 + k], o));
    }
  }
  // (e, Q): root's, then J ascending, then Sd ascending, replace iff Q_cand > Q (strict): the
  // first candidate attaining the maximum, if that maximum exceeds the root's Q
  const int src = qbest > q0 ? ibest : -1;
  // T_root <- ((T_root + T_j1) + T_j2 ...) + t_s1 ...   elementwise fp64, exactly this order
  double* Tr = M.T + (size_t)root * P.Dt;
  for (int d = lane; d < P.Dt; d += 32) {
    double acc = Tr[d];
    for (uint32_t i = 1; i < mcnt; ++i) acc = __dadd_rn(acc, M.T[(size_t)mem[i] * P.Dt + d]);
    for (uint32_t k = 0; k < dcnt; ++k) acc = __dadd_rn(acc, trk[(size_t)dets[k] * P.Dt + d]);
    Tr[d] = acc;
  }
  __syncwarp();
  if (P.Dt > 0) {
    const double tt = dot_pin_reg(Tr, Tr, P.Dt);
    if (lane == 0) M.TT[root] = tt;
  }
  if (src >= 0) {
    const float4* e = (const float4*)((uint32_t)src < mcnt ? M.E + (size_t)mem[src] * P.Df
                                                           : wb.emb + (fo + dets[src - mcnt]) * P.Df);
    float4* ed = (float4*)(M.E + (size_t)root * P.Df);
    for (int d4 = lane; d4 < P.Df / 4; d4 += 32) ed[d4] = e[d4];
  }
  // members: key lists of physical labels other than the survivor's were captured by K6 as
  // relabel segments; reset them, kill J (same lane per member: read before the kill)
  for (uint32_t i = lane; i < mcnt; i += 32) {
    const uint32_t m = mem[i];
    const uint32_t pm = M.phys_of[m];
    if (pm != L) {
      M.lst_len[pm] = 0;
      M.lst_cap[pm] = 0;
    }
    if (i >= 1) {
      M.alive[m] = 0;
      M.phys_of[m] = U32_EMPTY;
    }
  }
  if (lane == 0) {
    M.obs[root] = obs;
    M.last_seen[root] = F.frame_id;
    M.q[root] = src >= 0 ? qbest : q0;
    M.vcount[root] = X.tg_vbase[t];
    M.phys_of[root] = L;
    M.id_of[L] = root;
  }
  if (lane < 6) M.aabb[(size_t)root * 6 + lane] = ab[lane];
}

// Fast path (up to 32 members + detections, Dt <= 512): a few dependent memory round trips —
// descriptors; member / detection ids; their attributes and T / t rows together; the embedding
// copy — with T_root's sums and dot_pin(T, T) kept in registers (same lane / element order as
// dot_pin_reg: lane l holds d = l, l + 32, ... ascending).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// 1-D TMA: a bulk global -> shared copy completing on a shared-memory mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst), b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT;\n\t}" ::"r"(b),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ unsigned long long g_tgstep[8];   // DISC_S2PROF (-DTG_PROF): fast-path target sub-step time sums
#ifdef TG_PROF
#define TG_STEP(i)                                                          \
  do {                                                                      \
    unsigned long long t_;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    if (i >= 0 && lane == 0) atomicAdd(&g_tgstep[i], t_ - tg_t);          \
    tg_t = t_;                                                              \
  } while (0)
#else
#define TG_STEP(i) do { } while (0)
#endif
// stg: this warp's shared staging area for `rows` tracking rows and an embedding row, filled by 1-D
// TMA bulk copies completing on the mbarrier `bar` (phase ph) (nullptr: register path)
__device__ __forceinline__ void apply_target_warp(int t, int f, const FrameDesc& F, const WinBufs& wb,
                                                  const MapState& M, const FrameScratch& X, const Params& P, int sem,
                                                  double* stg, int rows, uint64_t* bar, uint32_t& ph) {
  const int lane = threadIdx.x & 31;
  unsigned long long tg_t = 0;
  TG_STEP(-1);
  const size_t fo = (size_t)f * wb.SMAX;
  const double* trk = wb.trk + fo * P.Dt;
  const int kind = X.tg_kind[t];
  const uint32_t root = X.tgt_root[t], L = X.tgt_phys[t];
  const uint32_t mcnt = X.tg_mcnt[t], dcnt = X.tg_dcnt[t];
  const int64_t vbase = X.tg_vbase[t];
  const int Dt = P.Dt, Df = P.Df;
  if (mcnt + dcnt > 32 || Dt > 512) {
    apply_target_warp_general(t, f, F, wb, M, X, P, sem);
    return;
  }
  const uint32_t n = mcnt + dcnt;
  DBOUND(root < (uint32_t)M.IMAX && (kind == 1 || L < (uint32_t)M.IMAX), M.err);
  // candidate of this lane: members (ids ascending) then detections (s ascending); K6 wrote them
  // side by side (tg_cand), one read with the descriptors
  const bool is_mem = (uint32_t)lane < mcnt, is_det = !is_mem && (uint32_t)lane < n;
  const uint32_t cid = (is_mem || is_det) ? X.tg_cand[t * 32 + lane] : 0u;
  DBOUND(!is_mem || cid < (uint32_t)M.IMAX, M.err);
  DBOUND(!is_det || cid < (uint32_t)F.S, M.err);

  TG_STEP(0);
  // attributes of the candidate
  int obs = 0;
  float qi = -INFINITY;
  uint32_t pm = U32_EMPTY;
  int32_t ab[6] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN};
  if (is_mem) {
    obs = M.obs[cid];
    qi = M.q[cid];
    pm = M.phys_of[cid];
    for (int k = 0; k < 6; ++k) ab[k] = M.aabb[(size_t)cid * 6 + k];
  } else if (is_det) {
    obs = 1;
    qi = wb.qf[(fo + cid) * 6 + 4];
    for (int k = 0; k < 6; ++k) ab[k] = wb.daabb[(fo + cid) * 6 + k];
  }
  TG_STEP(1);
  // T sums, pinned order: T_root (new instance: t_s1) then J ascending then Sd ascending
  double acc[16];
  const int nt = (Dt + 31) / 32;
  const uint32_t cid0 = __shfl_sync(0xffffffffu, cid, 0);   // (outside the lane-dependent branches)
  // new instance: its embedding row goes to shared memory with the tracking rows' first batch
  // (staged path; no registers held across the sums), else it is copied at the end
  const int D4 = Df / 4;
  float4* stg_e = stg ? (float4*)(stg + (size_t)rows * Dt) : nullptr;
  const bool e_stg = stg && kind == 1 && sem;
  if (stg) {
    // the candidates' rows (candidate 0 = the base: T_root = T of mem[0], the min id, or t_s1),
    // `rows` at a time: lane i copies candidate i's row with one bulk copy (the TMA engine moves
    // them, not the warp's load slots), one round trip per batch; summed in the pinned order from
    // shared memory
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    const uint32_t rb = (uint32_t)Dt * 8u;   // bytes per row
    for (uint32_t i0 = 0; i0 < n; i0 += (uint32_t)rows) {
      const uint32_t nb = min((uint32_t)rows, n - i0);
      fence_proxy_async_smem();   // (this warp's reads of the previous batch before the async writes)
      __syncwarp();
      const bool e_now = e_stg && i0 == 0;
      if (lane == 0) mbar_expect(bar, nb * rb + (e_now ? (uint32_t)Df * 4u : 0u));
      __syncwarp();
      if ((uint32_t)lane >= i0 && (uint32_t)lane < i0 + nb) {
        const uint32_t i = (uint32_t)lane;
        DBOUND(i - i0 < (uint32_t)rows, M.err);
        const double* row = (kind == 0 && i < mcnt) ? M.T + (size_t)cid * Dt : trk + (size_t)cid * Dt;
        bulk_g2s(stg + (size_t)(i - i0) * Dt, row, rb, bar);
      }
      if (e_now && lane == 31) bulk_g2s(stg_e, wb.emb + (fo + cid0) * Df, (uint32_t)Df * 4u, bar);
      mbar_wait(bar, ph);
      ph ^= 1u;
      for (uint32_t b = 0; b < nb; ++b) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int d = lane + 32 * k;
          if (k < nt && d < Dt) acc[k] = (i0 + b == 0) ? stg[d] : __dadd_rn(acc[k], stg[(size_t)b * Dt + d]);
        }
      }
      __syncwarp();
    }
  } else {
    const uint32_t first = 1;   // candidate 0 is the base: T_root (= mem[0], the min id) or t_s1
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int d = lane + 32 * k;
      acc[k] = 0.0;
      if (k < nt && d < Dt) {
        if (kind == 1) acc[k] = trk[(size_t)cid0 * Dt + d];
        else acc[k] = M.T[(size_t)root * Dt + d];
      }
    }
    for (uint32_t i = first; i < n; ++i) {
      const uint32_t id = __shfl_sync(0xffffffffu, cid, i);
      const double* row = i < mcnt ? M.T + (size_t)id * Dt : trk + (size_t)id * Dt;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int d = lane + 32 * k;
        if (k < nt && d < Dt) acc[k] = __dadd_rn(acc[k], row[d]);
      }
    }
  }
  TG_STEP(2);
  double tt = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int d = lane + 32 * k;
    if (k < nt && d < Dt) {
      M.T[(size_t)root * Dt + d] = acc[k];
      tt = __fma_rn(acc[k], acc[k], tt);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) tt = __dadd_rn(tt, __shfl_xor_sync(0xffffffffu, tt, o));
  // obs, aabb: warp reductions; (e, Q): the first candidate after the base with the maximum Q,
  // if it beats the base's (strict replacement in the pinned order)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    obs += __shfl_xor_sync(0xffffffffu, obs, o);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      ab[k] = min(ab[k], __shfl_xor_sync(0xffffffffu, ab[k], o));
      ab[3 + k] = max(ab[3 + k], __shfl_xor_sync(0xffffffffu, ab[3 + k], o));
    }
  }
  const float q0 = __shfl_sync(0xffffffffu, qi, 0);
  int src = -1;
  float qnew = q0;
  if (kind == 0) {
    const bool cand = (uint32_t)lane >= 1 && (uint32_t)lane < n;
    float qm = cand ? qi : -INFINITY;
#pragma unroll
    for (int o = 16; o; o >>= 1) qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
    const unsigned hit = __ballot_sync(0xffffffffu, cand && qi == qm);
    if (hit && qm > q0) { src = __ffs(hit) - 1; qnew = qm; }
  }
  const bool has_e = kind == 1 ? (sem && q0 >= 0.f) : src >= 0;
  const uint32_t sid = __shfl_sync(0xffffffffu, cid, src >= 0 ? src : 0);
  const float4* es = kind == 1 ? (const float4*)(wb.emb + (fo + sid) * Df)
                               : ((uint32_t)src < mcnt ? (const float4*)(M.E + (size_t)sid * Df)
                                                       : (const float4*)(wb.emb + (fo + sid) * Df));
  float4* ed = (float4*)(M.E + (size_t)root * Df);
  if (kind == 1) {
    const float4* src = stg_e ? stg_e : (const float4*)(wb.emb + (fo + cid0) * Df);
    for (int d4 = lane; d4 < D4; d4 += 32) ed[d4] = has_e ? src[d4] : make_float4(0.f, 0.f, 0.f, 0.f);
  } else if (has_e) {
    for (int d4 = lane; d4 < Df / 4; d4 += 32) ed[d4] = es[d4];
  }
  TG_STEP(3);
  if (kind == 0 && is_mem) {   // members: lists of other physical labels reset, J killed
    if (pm != L) {
      M.lst_len[pm] = 0;
      M.lst_cap[pm] = 0;
    }
    if (lane >= 1) {
      M.alive[cid] = 0;
      M.phys_of[cid] = U32_EMPTY;
    }
  }
  if (lane == 0) {
    if (kind == 1) {
      M.alive[root] = 1;
      M.phys_of[root] = root;
      M.id_of[root] = root;
      M.vcount[root] = 0;
      M.obs[root] = 1;
      M.q[root] = q0;
      M.lst_len[root] = 0;
    } else {
      M.obs[root] = obs;
      M.q[root] = qnew;
      M.vcount[root] = vbase;
      M.phys_of[root] = L;
      M.id_of[L] = root;
    }
    M.last_seen[root] = F.frame_id;
    if (Dt > 0) M.TT[root] = tt;
  }
  if (lane < 6) M.aabb[(size_t)root * 6 + lane] = ab[lane];
  TG_STEP(4);
}

// tagn != 0: frame f+1 was counted speculatively against the map before this update (into Cn; its
// pairs chained on their slots under tagn): every label this update adds to (+1) or tombstones on (-1)
// a slot corrects c_{s,label} of each of frame f+1's pairs (s, key) on that slot, so that frame f+1's
// counts are exactly those its own lookup after this update would find (aggregated per CTA in shared
// memory, added to Cn at the end).
constexpr int DT_CT = 1024;   // per-CTA correction table slots
#ifndef K7_DYN
#define K7_DYN 0
#endif
// Frame pf's pair records, home slots and slot-chain words pulled into L2 by every warp of the grid
// (one pair per lane per step): the speculative counting of frame pf runs two phases later against a
// 2 GB table whose random slot reads otherwise dominate it
__device__ __forceinline__ void s2_prefetch_frame(int pf, const WinBufs& wb, const MapState& M) {
  const uint32_t np = min(__ldcg(&wb.npairs[pf]), (uint32_t)wb.PMAX);
  const size_t fo = (size_t)pf * wb.PMAX;
  const uint32_t hmask = (uint32_t)(M.MC - 1);
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x, gn = gridDim.x * blockDim.x;
  for (uint32_t i = gt; i < np; i += gn) {
    if ((i & 31) == 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wb.pinfo + fo + i));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wb.pkey + fo + i + 16));
    }
    const unsigned long long key = __ldcg(&wb.pkey[fo + i]);
    const uint32_t h = (uint32_t)mix64(key) & hmask;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(M.slots + h));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(M.slh + h));
  }
}

#ifndef K7_PREFETCH
#define K7_PREFETCH 0   // (measured no net gain: -3 us counting, +2.5 us apply) frame f+2's map lines into L2 during frame f's apply
#endif
#ifndef K7_LOCKSTEP
#define K7_LOCKSTEP 1   // the two items of a lane in lockstep (0: one after the other, round 1)
#endif
#ifndef K7_TGT_NOCHUNK
#define K7_TGT_NOCHUNK 0
#endif
__device__ __forceinline__ void s2_apply(int f, const FrameDesc& F, const WinBufs& wb, const MapState& M,
                                         const FrameScratch& X, const Params& P, int sem,
                                         const CTab& Cn, uint32_t tagn = 0, int prof = 0, int pfn = -1) {
  const int lane = threadIdx.x & 31;
  unsigned long long ta0 = 0;
  auto amark = [&](int i) {   // DISC_S2PROF: sub-step end times (max over the warps, this frame)
    if (!prof || lane != 0) return;
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    if (i < 0) ta0 = t_;
    else atomicMax(&g_approf[i], t_ - ta0);
  };
  amark(-1);
  // targets spread over the CTAs first (warp w of CTA b takes target w * G + b), so no CTA holds
  // them all and the items are shared out evenly
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x, nw = gridDim.x * (blockDim.x >> 5);
  const int ntgt = *X.ntgt;
  // per-detection / per-target routing in shared memory (the association's bytes are free now)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* to_s = (unsigned long long*)smem_raw;   // [SMAX] list offsets
  int32_t* dt_s = (int32_t*)(to_s + wb.SMAX);                  // [SMAX] detection -> target
  uint32_t* tp_s = (uint32_t*)(dt_s + wb.SMAX);                // [SMAX] target -> physical label
  uint32_t* tb_s = tp_s + wb.SMAX;                             // [SMAX] target -> list length before
  for (int i = threadIdx.x; i < F.S; i += blockDim.x) dt_s[i] = X.det_target[i];
  for (int t = threadIdx.x; t < ntgt; t += blockDim.x) {
    tp_s[t] = X.tgt_phys[t];
    tb_s[t] = X.tgt_base[t];
    to_s[t] = X.tg_newoff[t];
  }
  uint32_t dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  // the correction table at the end of the dynamic shared memory
  const uint32_t dtb = (dyn - DT_CT * 12u) & ~15u;
  unsigned long long* dk = (unsigned long long*)(smem_raw + dtb);
  uint32_t* dc = (uint32_t*)(dk + DT_CT);
  if (tagn)
    for (int i = threadIdx.x; i < DT_CT; i += blockDim.x) { dk[i] = KEY_EMPTY; dc[i] = 0; }
  __syncthreads();
  amark(0);
  auto dt_add = [&](unsigned long long code, uint32_t add) {
    uint32_t h = (uint32_t)mix64(code) & (DT_CT - 1);
    for (int probe = 0; probe < 32; ++probe) {
      unsigned long long k = dk[h];
      if (k == KEY_EMPTY) {
        k = atomicCAS(&dk[h], KEY_EMPTY, code);
        if (k == KEY_EMPTY) k = code;
      }
      if (k == code) {
        atomicAdd(&dc[h], add);
        return;
      }
      h = (h + 1) & (DT_CT - 1);
    }
    count_add(Cn, code, add, M.err);
  };
  // shared staging (TMA bulk copies) for warp 0's tracking rows: the targets of a frame (a few dozen,
  // fewer than the CTAs) are each warp 0 of one CTA; up to 32 rows (a fast-path target's candidates
  // in one round trip) as far as the bytes between the routing and the correction tables allow
  double* stg = nullptr;
  uint64_t* bar = nullptr;
  int rows = 0;
  uint32_t ph = 0;
  {
    const size_t base = ((size_t)wb.SMAX * 20 + 127) & ~(size_t)127;
    const size_t room = dtb > base + 128 + (size_t)P.Df * 4 ? dtb - base - 128 - (size_t)P.Df * 4 : 0;
    rows = P.Dt > 0 ? (int)min((size_t)32, room / ((size_t)P.Dt * 8)) : 0;
    if (P.Dt > 0 && (P.Dt & 1) == 0 && (P.Df & 3) == 0 && rows >= 4 && (threadIdx.x >> 5) == 0) {
      bar = (uint64_t*)(smem_raw + base);
      stg = (double*)(smem_raw + base + 128);
      if (lane == 0) mbar_init(bar);
      __syncwarp();
    }
  }
  for (int t = gw; t < ntgt; t += nw) {
    unsigned long long t0_ = 0, t1_;
    if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0_));
    apply_target_warp(t, f, F, wb, M, X, P, sem, stg, rows, bar, ph);
    if (prof) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1_));
      if (lane == 0) {
        atomicAdd(&g_tgprof[0], t1_ - t0_);
        atomicMax(&g_tgprof[1], t1_ - t0_);
        atomicAdd(&g_tgprof[2], 1ull);
        const uint32_t n = X.tg_kind[t] ? 0u : min(33u, X.tg_mcnt[t] + X.tg_dcnt[t]);   // 0: new instance
        const int b = n == 0 ? 0 : n <= 2 ? 1 : n <= 4 ? 2 : n <= 8 ? 3 : n <= 16 ? 4 : n <= 32 ? 5 : 6;
        atomicAdd(&g_tghist[b], t1_ - t0_);
        atomicAdd(&g_tghist[8 + b], 1ull);
        atomicMax(&g_tghist[16 + b], t1_ - t0_);
      }
    }
  }
  amark(1);
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const uint32_t nrel = *X.nrel;
  const uint32_t nmove = X.tg_mvoff[ntgt];
  const uint32_t total = np + nrel + nmove;
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // (cheap; counted always, printed under DISC_S2PROF)
    atomicAdd(&g_s2items[0], (unsigned long long)np);
    atomicAdd(&g_s2items[1], (unsigned long long)nrel);
    atomicAdd(&g_s2items[2], (unsigned long long)nmove);
    atomicAdd(&g_s2items[3], (unsigned long long)ntgt);
  }
  const size_t fo = (size_t)f * wb.PMAX;
  const size_t f1o = fo + wb.PMAX;   // frame f+1's pair records (tagn)
  const int nseg = *X.nseg;
  int delta = 0;
  // items: frame pairs (inserts), relabel items, entries of lists K6 moved (copies), two items per
  // lane with their record loads issued together.  The pair items (the bulk: every unique (s, key)
  // of the frame, most already members) are split statically over the warps in 64-item blocks; the
  // relabel / copy items (uneven) come in 64-item chunks from a counter.  (All chunks from one
  // counter serialised ~1.5 k atomics per H frame on one L2 address.)
  const uint32_t npb = (np + 63) / 64;   // pair blocks
  // block b goes to warp (b + ntgt) mod nw: the target warps (gw < ntgt) get one only when there are
  // more blocks than other warps
  uint32_t sblk = ((uint32_t)gw + (uint32_t)nw - (uint32_t)min(ntgt, nw)) % (uint32_t)nw;
  // K7_DYN 0: the relabel / copy blocks (items np .. total) follow the pair blocks in the same static
  // round robin (no shared counter: every warp's one atomic on it serialised ~1.6 k atomics per frame
  // on one L2 address); 1: they come in 64-item chunks from X.work
  const uint32_t nbt = npb + (K7_DYN ? 0u : (nrel + nmove + 63) / 64);
  for (;;) {
    uint32_t base = 0;
    const bool stat = sblk < npb;   // a static pair block: its items past np are nobody's
    if (stat) {
      base = sblk * 64u;
      sblk += (uint32_t)nw;
    } else if (!K7_DYN) {
      if (sblk >= nbt) break;
      base = np + (sblk - npb) * 64u;
      sblk += (uint32_t)nw;
    } else {
      if (K7_TGT_NOCHUNK && gw < ntgt) break;   // (target warps leave the uneven items to the others)
      if (lane == 0) base = atomicAdd(X.work, 64u);
      base = __shfl_sync(0xffffffffu, base, 0) + npb * 64u;
      if (base >= npb * 64u + nrel + nmove) break;
      base -= (npb * 64u - np);   // -> the item index space: relabel items start at np
    }
    uint32_t itq[2], sq[2], slotq[2];
    uint2 plq[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {   // the pair records of both items first
      itq[q] = base + 32 * q + lane;
      sq[q] = 0; slotq[q] = U32_EMPTY; plq[q] = make_uint2(U32_EMPTY, U32_EMPTY);
      if (itq[q] < np) {
        sq[q] = wb.pinfo[fo + itq[q]];
        slotq[q] = wb.pms[fo + itq[q]];
        plq[q] = wb.plab[fo + itq[q]];
      }
    }
#if K7_LOCKSTEP
    // both items of the lane advance together, stage by stage, so that their independent memory
    // operations (records, slot reads, label CAS / tombstone, list appends, corrections) are in
    // flight at once instead of one item's chain after the other's
    int kd[2], tq[2], eq[2], tc[2];   // kind (0 none, 1 insert, 2 relabel), target, insert cell, tomb cell
    uint32_t Lq[2], Lo[2], sl[2];
    bool ins[2], tomb[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {   // classify; relabel items: their slot from the old label's list
      const uint32_t it = itq[q];
      kd[q] = 0; tq[q] = -1; eq[q] = -1; tc[q] = -1; Lq[q] = U32_EMPTY; Lo[q] = U32_EMPTY; sl[q] = U32_EMPTY;
      ins[q] = false; tomb[q] = false;
      if (it < np) {
        DBOUND(sq[q] < (uint32_t)F.S, M.err);
        const int t = dt_s[sq[q]];
        DBOUND(t < ntgt, M.err);
        if (t >= 0) {
          const uint32_t L = tp_s[t];
          const uint32_t slot = slotq[q];
          DBOUND(slot == U32_EMPTY || slot < M.MC, M.err);
          if (!(slot != U32_EMPTY && (plq[q].x == L || plq[q].y == L))) {   // else: already a member
            kd[q] = 1; tq[q] = t; Lq[q] = L; sl[q] = slot;
            // first EMPTY cell as the lookup saw it, when it saw the whole inline list (at most one
            // label): a CAS there without reading the slot again; any other outcome than EMPTY or L
            // takes the general insert
            if (slot != U32_EMPTY && plq[q].y == U32_EMPTY) eq[q] = plq[q].x == U32_EMPTY ? 0 : 1;
          }
        }
      } else if (!stat && it < np + nrel) {
        const uint32_t r = it - np;
        int lo = 0, hi = nseg - 1;   // last segment with seg_off <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (X.seg_off[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        kd[q] = 2;
        tq[q] = X.seg_tgt[lo];
        DBOUND(lo >= 0 && lo < nseg && tq[q] >= 0 && tq[q] < ntgt, M.err);
        DBOUND(X.seg_base[lo] + (r - X.seg_off[lo]) < M.ARENA, M.err);
        Lq[q] = tp_s[tq[q]];
        Lo[q] = X.seg_phys[lo];
        sl[q] = M.arena[X.seg_base[lo] + (r - X.seg_off[lo])];
        DBOUND(sl[q] < M.MC, M.err);
      } else if (!stat && it < total) {
        const uint32_t r = it - np - nrel;
        int lo = 0, hi = ntgt - 1;   // last target with tg_mvoff <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (X.tg_mvoff[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t i = r - X.tg_mvoff[lo];
        DBOUND(X.tg_newoff[lo] + i < M.ARENA && X.tg_movesrc[lo] + i < M.ARENA, M.err);
        M.arena[X.tg_newoff[lo] + i] = M.arena[X.tg_movesrc[lo] + i];
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {   // keys absent at lookup time (new this frame or since)
      if (kd[q] == 1 && sl[q] == U32_EMPTY) {
        bool created = false;
        sl[q] = map_insert_key_c(M, wb.pkey[fo + itq[q]], &created);
        if (sl[q] == U32_EMPTY) kd[q] = 0;
        else if (created) eq[q] = 0;
      }
    }
    SlotV sv[2];
#pragma unroll
    for (int q = 0; q < 2; ++q)   // relabel items: one read of each slot's inline labels
      if (kd[q] == 2) sv[q] = slot_load(M, sl[q]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {   // relabel: insert cell (first EMPTY, L absent), tomb cell (Lo's)
      if (kd[q] != 2) continue;
      bool present = false, full = true;
      int e = -1, c = -1;
#pragma unroll
      for (int i = 0; i < INLINE_LABELS; ++i) {
        const uint32_t v = sv[q].lab[i];
        if (!full) continue;   // (labels occupy a prefix: nothing after the first EMPTY)
        if (v == U32_EMPTY) { full = false; e = i; continue; }
        if (v == Lq[q]) present = true;
        if (v == Lo[q]) c = i;
      }
      eq[q] = present ? -2 : (full ? -1 : e);   // -2: L already there; -1: general insert
      tc[q] = c >= 0 ? c : (full ? -1 : -2);    // -2: Lo not on the key; -1: general tombstone
    }
    uint32_t old[2] = {U32_EMPTY, U32_EMPTY};
#pragma unroll
    for (int q = 0; q < 2; ++q)   // the insert CASes of both items, then the tombstones
      if (kd[q] != 0 && eq[q] >= 0) old[q] = atomicCAS(&M.slots[sl[q]].lab[eq[q]], U32_EMPTY, Lq[q]);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (kd[q] == 2 && tc[q] >= 0) { atomicExch(&M.slots[sl[q]].lab[tc[q]], LAB_TOMB); tomb[q] = true; }
#pragma unroll
    for (int q = 0; q < 2; ++q) {   // outcomes; the general routines for everything else
      if (kd[q] == 0) continue;
      if (eq[q] >= 0) ins[q] = old[q] == U32_EMPTY ? true : (old[q] == Lq[q] ? false : label_insert(M, sl[q], Lq[q]));
      else if (eq[q] == -1) ins[q] = label_insert(M, sl[q], Lq[q]);
      if (kd[q] == 2 && tc[q] == -1) tomb[q] = label_tomb(M, sl[q], Lo[q]);
      delta += (ins[q] ? 1 : 0) - (tomb[q] ? 1 : 0);
    }
    // append the new (target, slot) entries to the targets' lists (warp-aggregated positions; K6
    // reserved the room): both items' atomics, then both items' stores
    unsigned peers[2];
    uint32_t pb[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int tn = ins[q] ? tq[q] : -1;
      peers[q] = __match_any_sync(0xffffffffu, tn);
      pb[q] = 0;
      if (tn >= 0 && lane == __ffs(peers[q]) - 1) pb[q] = atomicAdd(&X.tgt_stage[tn], (uint32_t)__popc(peers[q]));
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int tn = ins[q] ? tq[q] : -1;
      const uint32_t b = __shfl_sync(0xffffffffu, pb[q], __ffs(peers[q]) - 1);
      if (tn >= 0) {
        DBOUND(to_s[tn] + tb_s[tn] + b + __popc(peers[q] & ((1u << lane) - 1u)) < M.ARENA, M.err);
        M.arena[to_s[tn] + tb_s[tn] + b + __popc(peers[q] & ((1u << lane) - 1u))] = sl[q];
      }
    }
    if (tagn) {   // count corrections of frame f+1 (warp-aggregated per (s, label) and sign)
      uint32_t pi[2];
      unsigned long long v[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        v[q] = 0;
        if (ins[q] || tomb[q]) v[q] = __ldcg(&M.slh[sl[q]]);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) pi[q] = (ins[q] || tomb[q]) && (uint32_t)(v[q] >> 32) == tagn ? (uint32_t)v[q] : U32_EMPTY;
      while (__any_sync(0xffffffffu, pi[0] != U32_EMPTY || pi[1] != U32_EMPTY)) {
        unsigned long long sh[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) DBOUND(pi[q] == U32_EMPTY || pi[q] < (uint32_t)wb.PMAX, M.err);
#pragma unroll
        for (int q = 0; q < 2; ++q) sh[q] = pi[q] != U32_EMPTY ? (unsigned long long)__ldcg(&wb.pinfo[f1o + pi[q]]) << 32 : 0;
        uint32_t nx[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) nx[q] = pi[q] != U32_EMPTY ? __ldcg(&wb.pnext[f1o + pi[q]]) : U32_EMPTY;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const unsigned long long ci = pi[q] != U32_EMPTY && ins[q] ? sh[q] | Lq[q] : KEY_EMPTY;
          const unsigned long long ct = pi[q] != U32_EMPTY && tomb[q] ? sh[q] | Lo[q] : KEY_EMPTY;
          const unsigned pa = __match_any_sync(0xffffffffu, ci);
          if (ci != KEY_EMPTY && lane == __ffs(pa) - 1) dt_add(ci, (uint32_t)__popc(pa));
          const unsigned pt = __match_any_sync(0xffffffffu, ct);
          if (ct != KEY_EMPTY && lane == __ffs(pt) - 1) dt_add(ct, (uint32_t)(-__popc(pt)));
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) pi[q] = nx[q];
      }
    }
#else
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t it = itq[q];
      int tnew = -1;
      uint32_t snew = 0;
      uint32_t dslot = U32_EMPTY;   // the slot whose labels changed (tagn)
      uint32_t dLi = U32_EMPTY, dLt = U32_EMPTY;   // label added / tombstoned on it
      if (it < np) {
        const int t = dt_s[sq[q]];
        if (t >= 0) {
          const uint32_t L = tp_s[t];
          uint32_t slot = slotq[q];
          if (!(slot != U32_EMPTY && (plq[q].x == L || plq[q].y == L))) {   // else: already a member
            // first EMPTY cell as the lookup saw it, when it saw the whole inline list (at most one
            // label): a CAS there, without reading the slot again; any other outcome than EMPTY or
            // L takes the general insert
            int e = -1;
            if (slot == U32_EMPTY) {
              bool created = false;
              slot = map_insert_key_c(M, wb.pkey[fo + it], &created);
              if (created) e = 0;
            } else if (plq[q].y == U32_EMPTY) {
              e = plq[q].x == U32_EMPTY ? 0 : 1;
            }
            if (slot != U32_EMPTY) {
              bool ins;
              if (e >= 0) {
                const uint32_t old = atomicCAS(&M.slots[slot].lab[e], U32_EMPTY, L);
                ins = old == U32_EMPTY ? true : (old == L ? false : label_insert(M, slot, L));
              } else {
                ins = label_insert(M, slot, L);
              }
              if (ins) { tnew = t; snew = slot; delta++; dslot = slot; dLi = L; }
            }
          }
        }
      } else if (!stat && it < np + nrel) {
        const uint32_t r = it - np;
        int lo = 0, hi = nseg - 1;   // last segment with seg_off <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (X.seg_off[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        const int t = X.seg_tgt[lo];
        const uint32_t L = tp_s[t];
        const uint32_t slot = M.arena[X.seg_base[lo] + (r - X.seg_off[lo])];
        if (label_insert(M, slot, L)) { tnew = t; snew = slot; delta++; dLi = L; }
        const uint32_t Lo = X.seg_phys[lo];
        if (label_tomb(M, slot, Lo)) { delta--; dLt = Lo; }
        dslot = slot;
      } else if (!stat && it < total) {
        const uint32_t r = it - np - nrel;
        int lo = 0, hi = ntgt - 1;   // last target with tg_mvoff <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (X.tg_mvoff[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t i = r - X.tg_mvoff[lo];
        M.arena[X.tg_newoff[lo] + i] = M.arena[X.tg_movesrc[lo] + i];
      }
      // append the new (target, slot) entries to the targets' lists (warp-aggregated positions;
      // K6 reserved the room)
      const unsigned peers = __match_any_sync(0xffffffffu, tnew);
      const int leader = __ffs(peers) - 1;
      uint32_t pb = 0;
      if (tnew >= 0 && lane == leader) pb = atomicAdd(&X.tgt_stage[tnew], (uint32_t)__popc(peers));
      pb = __shfl_sync(0xffffffffu, pb, leader);
      if (tnew >= 0) {
        const uint32_t pos = tb_s[tnew] + pb + __popc(peers & ((1u << lane) - 1u));
        M.arena[to_s[tnew] + pos] = snew;
      }
      if (tagn) {   // count corrections of frame f+1 (warp-aggregated per (s, label) and sign)
        uint32_t pi = U32_EMPTY;
        if (dslot != U32_EMPTY && (dLi != U32_EMPTY || dLt != U32_EMPTY)) {
          const unsigned long long v = __ldcg(&M.slh[dslot]);
          if ((uint32_t)(v >> 32) == tagn) pi = (uint32_t)v;
        }
        while (__any_sync(0xffffffffu, pi != U32_EMPTY)) {
          unsigned long long ci = KEY_EMPTY, ct = KEY_EMPTY;
          if (pi != U32_EMPTY) {
            const unsigned long long sh = (unsigned long long)__ldcg(&wb.pinfo[f1o + pi]) << 32;
            if (dLi != U32_EMPTY) ci = sh | dLi;
            if (dLt != U32_EMPTY) ct = sh | dLt;
            pi = __ldcg(&wb.pnext[f1o + pi]);
          }
          const unsigned pa = __match_any_sync(0xffffffffu, ci);
          if (ci != KEY_EMPTY && lane == __ffs(pa) - 1) dt_add(ci, (uint32_t)__popc(pa));
          const unsigned pt = __match_any_sync(0xffffffffu, ct);
          if (ct != KEY_EMPTY && lane == __ffs(pt) - 1) dt_add(ct, (uint32_t)(-__popc(pt)));
        }
      }
    }
#endif
  }
  amark(2);
  if (K7_PREFETCH && pfn >= 0) s2_prefetch_frame(pfn, wb, M);
#pragma unroll
  for (int o = 16; o; o >>= 1) delta += __shfl_xor_sync(0xffffffffu, delta, o);
  if (lane == 0 && delta) atomicAdd((unsigned long long*)&M.counters[2], (unsigned long long)(int64_t)delta);
  if (tagn) {   // the CTA's corrections into frame f+1's count table
    __syncthreads();
    for (int i = threadIdx.x; i < DT_CT; i += blockDim.x)
      if (dc[i]) count_add(Cn, dk[i], dc[i], M.err);
  }
  amark(3);
}

// While CTA 0 starts the association of frame f, CTAs 1.. evaluate the pinned fp64 visual gate
// (R15) of every (s, j) triple of the frame, warp per triple (the association keeps the geometric
// edges whose gate passed).  Same dot_pin_reg as the single-CTA path: the same bits.
// (on CTAs 1 .. gc)
__device__ __forceinline__ void s2_gate(int f, const WinBufs& wb, const MapState& M, const FrameScratch& X,
                                     const CTab& C, const Params& P, uint32_t gc) {
  const uint32_t ntr = min(__ldcg(C.ntrip), (uint32_t)X.TCAP);
  const size_t fo = (size_t)f * wb.SMAX;
  const double* trk = wb.trk + fo * P.Dt;
  const int lane = threadIdx.x & 31;
  const uint32_t nwc = blockDim.x >> 5;
  const uint32_t w = (blockIdx.x - 1) * nwc + (threadIdx.x >> 5), nw = gc * nwc;
  uint32_t done = 0;
  for (uint32_t t = w; t < ntr; t += nw) {
    const uint32_t s = __ldcg(&C.ts[t]), j = __ldcg(&M.id_of[__ldcg(&C.tj[t])]);
    const double TT = __ldcg(&M.TT[j]);
    const uint8_t tok = wb.tok[fo + s];
    const double dt = dot_pin_reg(trk + (size_t)s * P.Dt, M.T + (size_t)j * P.Dt, P.Dt);
    double cosv = -2.0;
    if (tok && TT > 0.0) cosv = __ddiv_rn(dt, __dsqrt_rn(TT));
    if (lane == 0) X.trip_gate[t] = cosv >= (double)P.tau_vis ? 1 : 0;
    ++done;
  }
  if (lane == 0 && done) {
    __threadfence();
    atomicAdd(X.gate_done, done);
  }
}

// While CTA 0 runs the association of frame f, the other CTAs look up frame f+1's keys
// speculatively (against the map before frame f's update): each kept pair's slot index, or
// U32_EMPTY, into pms.  Frame f+1's lookup re-reads the found slots (their labels may have changed;
// the slot of a key never does) and probes only the keys absent here.
__device__ __forceinline__ void s2_spec(int f, const WinBufs& wb, const MapState& M) {
  const uint32_t np = min(__ldcg(&wb.npairs[f]), (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  const uint32_t hmask = (uint32_t)(M.MC - 1);
  const int32_t* stf = wb.status + (size_t)f * wb.SMAX;
  const uint32_t nth = (gridDim.x - 1) * blockDim.x;   // CTAs 1..G-1
  constexpr int Q = 4;
  for (uint32_t b = (blockIdx.x - 1) * blockDim.x + threadIdx.x; b < np; b += Q * nth) {
    unsigned long long key[Q];
    uint32_t h[Q], res[Q];
    bool act[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t i = b + q * nth;
      act[q] = i < np && stf[__ldcg(&wb.pinfo[fo + i])] == 0;
      key[q] = act[q] ? __ldcg(&wb.pkey[fo + i]) : KEY_EMPTY;
      h[q] = (uint32_t)mix64(key[q]) & hmask;
      res[q] = U32_EMPTY;
    }
    for (uint32_t probe = 0; probe <= hmask; ++probe) {
      bool any = false;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (!act[q]) continue;
        const unsigned long long k = __ldcg(&M.slots[h[q]].key);
        if (k == key[q]) { res[q] = h[q]; act[q] = false; }
        else if (k == KEY_EMPTY) act[q] = false;
        else h[q] = (h[q] + 1) & hmask;
        any = any || act[q];
      }
      if (!any) break;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (b + q * nth < np) wb.pms[fo + b + q * nth] = res[q];
  }
}

// (DISC_S2_SPEC=0) the round-1 variant: only pull frame f+1's pair records and home slots into L2
__device__ __forceinline__ void s2_prefetch_hint(int f, const WinBufs& wb, const MapState& M) {
  const uint32_t np = min(__ldcg(&wb.npairs[f]), (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  const uint32_t hmask = (uint32_t)(M.MC - 1);
  const uint32_t n = gridDim.x - 1, b = blockIdx.x - 1;   // CTAs 1..G-1
  for (uint32_t i = b * blockDim.x + threadIdx.x; i < np; i += n * blockDim.x) {
    if ((i & 31) == 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wb.pinfo + fo + i));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wb.pms + fo + i));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wb.pkey + fo + i + 16));
    }
    const unsigned long long key = __ldcg(&wb.pkey[fo + i]);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(M.slots + ((uint32_t)mix64(key) & hmask)));
  }
}

// K7 tail, run in the next phase: list lengths and exact |V| of the frame's targets, insert counter,
// membership report fields
// (cta0: CTA 0 alone runs it, before the next association)
__device__ __forceinline__ void s2_finalize(int f, const MapState& M, const FrameScratch& X, bool cta0 = false) {
  const int ntgt = *X.ntgt;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    disc_frame_report& R = X.rep[f];
    R.live_memberships = M.counters[2];
    R.new_memberships = M.counters[2] - *X.live_before;
  }
  const int t0 = cta0 ? threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x;
  const int tn = cta0 ? blockDim.x : gridDim.x * blockDim.x;
  for (int t = t0; t < ntgt; t += tn) {
    const uint32_t add = X.tgt_stage[t];
    DBOUND(X.tgt_phys[t] < (uint32_t)M.IMAX && X.tgt_root[t] < (uint32_t)M.IMAX, M.err);
    M.lst_len[X.tgt_phys[t]] = X.tgt_base[t] + add;
    M.vcount[X.tgt_root[t]] += add;
    if (add) atomicAdd((unsigned long long*)&M.counters[5], (unsigned long long)add);
  }
}

size_t k6_layout_bytes(int S, int TC) { return K6Smem(S, TC).total; }

size_t k6_smem_bytes(int S, int TC) {
  // the association's layout; the lookup / apply phases reuse the same bytes
  return std::max(K6Smem(S, TC).total, (size_t)LK_CT * 12 + (size_t)S * 32 + 64);
}

void k6_prof_dump() {
  if (getenv("DISC_S2PROF")) {
    unsigned long long g[8];
    cudaMemcpyFromSymbol(g, g_s2prof, sizeof(g));
    fprintf(stderr, "s2 phase ns: lookup %llu assoc %llu apply %llu kernel span %llu (64 barriers x launches: %llu)\n", g[0], g[1], g[2], g[6], g[7]);
    unsigned long long c[8];
    cudaMemcpyFromSymbol(c, g_s2cta, sizeof(c));
    fprintf(stderr, "s2 per-frame CTA work maxima, summed: association (CTA 0) %llu, gate + next frame's counting %llu, apply %llu\n",
            c[4], c[5], c[6]);
    cudaMemcpyFromSymbol(c, g_s2items, 4 * sizeof(unsigned long long));
    fprintf(stderr, "s2 K7 items: pairs %llu relabels %llu moves %llu targets %llu\n", c[0], c[1], c[2], c[3]);
    unsigned long long lk[20];
    cudaMemcpyFromSymbol(lk, g_lkprof, sizeof(lk));
    for (int m = 0; m < 2; ++m) {
      const unsigned long long* c2 = lk + 10 * m;
      fprintf(stderr, "s2 %s (first CTA, thread 0): init %llu flush %llu | records %llu status+probes %llu slot-chains %llu labels %llu aggregate %llu wait-for-CTA %llu\n",
              m ? "speculative counting" : "lookup phase", c2[0], c2[2], c2[7], c2[3], c2[8], c2[4], c2[5], c2[6]);
    }
    cudaMemcpyFromSymbol(c, g_approf, 8 * sizeof(unsigned long long));
    fprintf(stderr, "s2 apply sub-steps (per-frame max end time, summed): routing %llu targets %llu items %llu flush %llu\n",
            c[4], c[5], c[6], c[7]);
    unsigned long long hh[24];
    cudaMemcpyFromSymbol(hh, g_tghist, sizeof(hh));
    fprintf(stderr, "s2 target time by candidates (sum ns / count / max ns):");
    const char* nm[7] = {"new", "<=2", "<=4", "<=8", "<=16", "<=32", ">32"};
    for (int b = 0; b < 7; ++b) fprintf(stderr, " %s %llu/%llu/%llu", nm[b], hh[b], hh[8 + b], hh[16 + b]);
    fprintf(stderr, "\n");
    cudaMemcpyFromSymbol(c, g_tgstep, 5 * sizeof(unsigned long long));
    fprintf(stderr, "s2 fast-path target steps (sums, -DTG_PROF): descriptors %llu attributes %llu rows+sums %llu e/Q %llu writes %llu\n",
            c[0], c[1], c[2], c[3], c[4]);
    cudaMemcpyFromSymbol(c, g_tgprof, 3 * sizeof(unsigned long long));
    fprintf(stderr, "s2 target warps: sum %llu max %llu count %llu\n", c[0], c[1], c[2]);
  }
  unsigned long long pl[4];
  cudaMemcpyFromSymbol(pl, g_s2place, sizeof(pl));
  fprintf(stderr, "s2 placement: %llu launches, %llu CTAs, %llu on SMs outside [0, grid)\n", pl[0], pl[1], pl[2]);
  unsigned long long h[16];
  cudaMemcpyFromSymbol(h, g_k6prof, sizeof(h));
  fprintf(stderr, "k6 phase ns (cumulative):");
  for (int i = 1; i < 14; ++i) fprintf(stderr, " %d:%llu", i - 1, h[i]);
  fprintf(stderr, "\n");
}

// Grid-wide barrier of the persistent stage-2 kernel (all CTAs co-resident: the grid is sized to
// the SMs K1 leaves free, one CTA per SM).  Monotonic counter, zeroed by K0 for the window.
__device__ __forceinline__ void grid_sync(uint32_t* bar, uint32_t target) {
  __syncthreads();   // the CTA's writes are ordered before thread 0's release (causality is cumulative)
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Stage 2 of a window: the frames' map updates in order, in one persistent launch.  Frame f's
// phases: K5 lookup (with frame f-1's K7 tail) | K6 association on CTA 0, the visual gate and the
// next frame's speculative work on CTAs 1.. | K7 apply, grid-synchronised.
//
// spec 2 (default): frame f+1 is counted during frame f's association (against the map before
// frame f's update) and frame f's K7 corrects those counts for every label it adds or tombstones on
// a key of frame f+1 (s2_apply), so frame f+1 needs no lookup phase: two barriers per frame instead
// of three.  spec 1: only frame f+1's slots are found early (its lookup re-reads them); 0: L2 hints.
// Frame f counts into table (f - f0) & 1 (Xc); Xn is the other one.
__device__ __forceinline__ void s2_frame(int f, int f0, int fe, const WinDesc& wd, const WinBufs& wb,
                                         const MapState& M, const FrameScratch& X, const Params& P, int sem,
                                         int spec, uint32_t& ep, int prof, uint32_t tag0) {
  const uint32_t G = gridDim.x;
  const FrameDesc& F = wd.f[f];
  const int p = (f - f0) & 1;
  const CTab Cc = ctab(X, p), Cn = ctab(X, p ^ 1);   // this frame's count table, the next one's
  const bool sp = spec >= 2 && f > f0 && G > 1;        // this frame was counted speculatively
  const bool spn = spec >= 2 && f + 1 < fe && G > 1;   // the next one will be
  auto probe = [&](int i) {   // DISC_S2PROF: phase end times on CTA 0 (profiling aid)
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      atomicAdd(&g_s2prof[i], t_ - g_s2prof[5]);
      g_s2prof[5] = t_;
    }
  };
  if (!sp) {
    if (K7_PREFETCH && spn) s2_prefetch_frame(f + 1, wb, M);   // (the window's first frame)
    s2_lookup(f, wb, M, X, Cc, spec == 1 && f > f0 && G > 1);
    if (f > f0) s2_finalize(f - 1, M, X);
    grid_sync(wb.s2bar, G * ++ep);
    probe(0);
  } else if (blockIdx.x == 0) {
    s2_finalize(f - 1, M, X, true);
    __syncthreads();
  }
  unsigned long long tph = 0;   // DISC_S2PROF: this CTA's work time per phase (max over the CTAs)
  auto cta_mark = [&](int slot) {
    if (!prof) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      if (slot >= 0) atomicMax(&g_s2cta[slot], t_ - tph);
      tph = t_;
    }
  };
  auto cta_fold = [&]() {   // (CTA 0 after a barrier: per-frame maxima into the sums)
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      for (int i = 0; i < 3; ++i) { g_s2cta[4 + i] += g_s2cta[i]; g_s2cta[i] = 0; }
      for (int i = 0; i < 4; ++i) { g_approf[4 + i] += g_approf[i]; g_approf[i] = 0; }
    }
  };
  cta_mark(-1);
  // spec 3: the gate on CTAs 1 .. gc (a triple per warp), frame f+1's counting on the others
  const uint32_t ntr_c = P.Dt > 0 && spec >= 3 ? min(__ldcg(Cc.ntrip), (uint32_t)X.TCAP) : 0u;
  const uint32_t gc = P.Dt > 0 ? min(max(1u, G / 4), max(1u, (ntr_c + 15) / 16)) : 0u;
  if (blockIdx.x == 0) {
    s2_assoc(f, F, wb, M, X, Cc, P, sem, f == f0, f == fe - 1);
    cta_mark(0);
  } else if (spec >= 3 && G > 2) {
    if (blockIdx.x <= gc) {
      if (P.Dt > 0) s2_gate(f, wb, M, X, Cc, P, gc);
    } else if (spn) {
      s2_lookup(f + 1, wb, M, X, Cn, false, 1 + gc, tag0 + (uint32_t)(f + 1));
    }
    cta_mark(1);
  } else {
    if (P.Dt > 0) s2_gate(f, wb, M, X, Cc, P, G - 1);
    if (spn) s2_lookup(f + 1, wb, M, X, Cn, false, 1, tag0 + (uint32_t)(f + 1));
    else if (f + 1 < fe) {
      if (spec) s2_spec(f + 1, wb, M);
      else s2_prefetch_hint(f + 1, wb, M);
    }
    cta_mark(1);
  }
  grid_sync(wb.s2bar, G * ++ep);
  probe(1);
  cta_fold();
  cta_mark(-1);
  // (frame f+2 is counted during frame f+1's association: its map lines into L2 now)
  s2_apply(f, F, wb, M, X, P, sem, Cn, spn ? tag0 + (uint32_t)(f + 1) : 0u, prof,
           spec >= 2 && f + 2 < fe && G > 1 ? f + 2 : -1);
  cta_mark(2);
  grid_sync(wb.s2bar, G * ++ep);
  probe(2);
  cta_fold();
}

__global__ void __launch_bounds__(K6_THREADS, 1) k_stage2(WinDesc wd, WinBufs wb, MapState M, FrameScratch X,
                                                        Params P, int sem, int prof, int spec, int f0, int fn,
                                                        uint32_t tag0) {
  const uint32_t G = gridDim.x;
  uint32_t ep = 0;
  unsigned long long t_k0 = 0;
  if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_k0));
    g_s2prof[5] = t_k0;
  }
  if (prof == 2) {   // DISC_S2PROF=2: cost of 64 empty grid barriers (profiling aid)
    for (int i = 0; i < 64; ++i) grid_sync(wb.s2bar, G * ++ep);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      atomicAdd(&g_s2prof[7], t_ - t_k0);
      g_s2prof[5] = t_;
    }
  }
  uint32_t sm_ = 0;
  if (threadIdx.x == 0) {   // this CTA's SM, published to stage 1 (on_reserved_sm); placement record
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
    atomicOr(&wb.s2sm[sm_ >> 5], 1u << (sm_ & 31));
    atomicAdd(&wb.s2sm[5], 1u);
    if (blockIdx.x == 0) atomicAdd(&g_s2place[0], 1ull);
    atomicAdd(&g_s2place[1], 1ull);
    if (sm_ >= G) atomicAdd(&g_s2place[2], 1ull);
  }
  const int fe = f0 + fn;   // frames [f0, fe) of the window (refine_active: one per launch)
  for (int f = f0; f < fe; ++f) s2_frame(f, f0, fe, wd, wb, M, X, P, sem, spec, ep, prof, tag0);
  if (fe > f0) s2_finalize(fe - 1, M, X);
  if (threadIdx.x == 0) {
    atomicSub(&wb.s2sm[5], 1u);
    atomicAnd(&wb.s2sm[sm_ >> 5], ~(1u << (sm_ & 31)));
  }
  if (prof && blockIdx.x == 0 && threadIdx.x == 0) {   // the kernel's own span (CTA 0)
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    atomicAdd(&g_s2prof[6], t_ - t_k0);
  }
}

// ------------------------------------------------------------------------------------------
// The key-hash-sharded map: the same three phases as k_stage2, one
// kernel each per frame and shard, so that the shards' partial results can be exchanged between
// them (kernel boundaries are the barriers; the exchange is NCCL across processes or device copies
// between the shards of one process).  Shard g holds the memberships of the keys it owns
// (owner = key_owner(key, G)) and a replica of the instance table, which every shard updates
// identically from identical (exchanged) inputs.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ FrameDesc meta_desc(const FrameMeta* meta, int f) {
  FrameDesc F{};
  F.S = meta[f].S;
  F.frame_id = meta[f].frame_id;
  return F;
}

__global__ void __launch_bounds__(K6_THREADS, 1) k_s2_lookup(int f, WinBufs wb, MapState M, FrameScratch X, Params P) {
  s2_lookup(f, wb, M, X, ctab(X, 0));
}

// X1 send side: this shard's partial (s, physical label, count) triples of frame f
__global__ void __launch_bounds__(512) k_trip_pack(FrameScratch X, uint32_t* out, int cap, int* err) {
  const uint32_t n = __ldcg(X.ntrip);
  if (n > (uint32_t)cap) {
    if (threadIdx.x == 0) { raise_err(err, DERR_TRIPLES); out[0] = 0; }
    return;
  }
  if (threadIdx.x == 0) out[0] = n;
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
    out[1 + 3 * t] = X.trip_s[t];
    out[2 + 3 * t] = X.trip_j[t];
    out[3 + 3 * t] = X.ctab_cnt[X.ctab_idx[t]];
  }
}

// X1 receive side: the other shards' partial triples added into this shard's count table (integer
// sums: every shard ends with the same (s, j) -> c_sj set, in any order)
__global__ void __launch_bounds__(256) k_trip_merge(FrameScratch X, const uint32_t* all, size_t stride, int G, int self,
                                                    int* err) {
  for (int g = 0; g < G; ++g) {
    if (g == self) continue;
    const uint32_t* b = all + (size_t)g * stride;
    const uint32_t n = b[0];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
      count_add(ctab(X, 0), ((uint64_t)b[1 + 3 * t] << 32) | b[2 + 3 * t], b[3 + 3 * t], err);
  }
}

__global__ void __launch_bounds__(K6_THREADS, 1) k_s2_assoc(int f, const FrameMeta* meta, WinBufs wb, MapState M,
                                                            FrameScratch X, Params P, int sem) {
  const FrameDesc F = meta_desc(meta, f);
  s2_assoc(f, F, wb, M, X, ctab(X, 0), P, sem);   // one CTA: it evaluates the visual gate of its candidates itself
}

__global__ void __launch_bounds__(K6_THREADS, 1) k_s2_apply(int f, const FrameMeta* meta, WinBufs wb, MapState M,
                                                            FrameScratch X, Params P, int sem) {
  const FrameDesc F = meta_desc(meta, f);
  s2_apply(f, F, wb, M, X, P, sem, ctab(X, 0));
}

// X2 send side: this shard's new memberships per target (own keys), its live count and the live
// count the association saw (report fields)
__global__ void k_add_pack(MapState M, FrameScratch X, int64_t* out, int smax) {
  const int ntgt = *X.ntgt;
  for (int t = threadIdx.x; t < smax; t += blockDim.x) out[t] = t < ntgt ? (int64_t)X.tgt_stage[t] : 0;
  if (threadIdx.x == 0) {
    out[smax] = M.counters[2];
    out[smax + 1] = *X.live_before;
  }
}

// K7 tail with the SUMMED adds: |V_root| grows by every shard's new memberships; the key lists
// (own keys) by this shard's
__global__ void k_s2_finalize_sum(int f, MapState M, FrameScratch X, const int64_t* all, int parts, size_t stride,
                                  int smax) {
  const int ntgt = *X.ntgt;
  auto sum = [&](int k) {   // fixed order over the shards' rows (integers: any order is exact)
    int64_t v = 0;
    for (int g = 0; g < parts; ++g) v += all[(size_t)g * stride + k];
    return v;
  };
  if (threadIdx.x == 0) {
    disc_frame_report& R = X.rep[f];
    R.live_memberships = sum(smax);
    R.new_memberships = sum(smax) - sum(smax + 1);
  }
  for (int t = threadIdx.x; t < ntgt; t += blockDim.x) {
    const uint32_t add = X.tgt_stage[t];
    M.lst_len[X.tgt_phys[t]] = X.tgt_base[t] + add;
    M.vcount[X.tgt_root[t]] += sum(t);
    if (add) atomicAdd((unsigned long long*)&M.counters[5], (unsigned long long)add);
  }
}

void launch_stage2_sharded_frame(int phase, int f, const FrameMeta* meta, const WinBufs& wb, const MapState& M,
                                 const FrameScratch& X, const Params& P, bool sem, int grid, cudaStream_t st) {
  const size_t sm6 = k6_smem_bytes(wb.SMAX, X.TCS);
  static size_t set_for = 0;
  if (set_for != sm6) {
    cudaFuncSetAttribute(k_s2_lookup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
    cudaFuncSetAttribute(k_s2_assoc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
    cudaFuncSetAttribute(k_s2_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
    set_for = sm6;
  }
  const int semi = sem ? 1 : 0;
  if (phase == 0) k_s2_lookup<<<grid, K6_THREADS, sm6, st>>>(f, wb, M, X, P);
  else if (phase == 1) k_s2_assoc<<<1, K6_THREADS, sm6, st>>>(f, meta, wb, M, X, P, semi);
  else k_s2_apply<<<grid, K6_THREADS, sm6, st>>>(f, meta, wb, M, X, P, semi);
  debug_check(st, phase == 0 ? "k_s2_lookup" : phase == 1 ? "k_s2_assoc" : "k_s2_apply", f);
}

void launch_trip_pack(const FrameScratch& X, uint32_t* out, int cap, int* err, cudaStream_t st) {
  k_trip_pack<<<1, 512, 0, st>>>(X, out, cap, err);
  debug_check(st, "k_trip_pack", -1);
}

void launch_trip_merge(const FrameScratch& X, const uint32_t* all, size_t stride, int G, int self, int* err,
                       cudaStream_t st) {
  k_trip_merge<<<16, 256, 0, st>>>(X, all, stride, G, self, err);
  debug_check(st, "k_trip_merge", -1);
}

void launch_add_pack(const MapState& M, const FrameScratch& X, int64_t* out, int smax, cudaStream_t st) {
  k_add_pack<<<1, 256, 0, st>>>(M, X, out, smax);
  debug_check(st, "k_add_pack", -1);
}

void launch_finalize_sum(int f, const MapState& M, const FrameScratch& X, const int64_t* all, int parts, size_t stride,
                         int smax, cudaStream_t st) {
  k_s2_finalize_sum<<<1, 256, 0, st>>>(f, M, X, all, parts, stride, smax);
  debug_check(st, "k_s2_finalize_sum", f);
}

// ------------------------------------------------------------------------------------------
// NEXT f2 (refine_active, reading R43): after frame f's update, the instance pairs of the frame's
// active set -- the instances its detections overlapped (the C triples' j, still alive) and its
// targets (component roots, new ids) -- that pass R36's test (the association's tau_geo / tau_vis)
// merge into their min id (R37), in rounds until no active pair qualifies (S:327 step (3)).
// One cooperative kernel per frame, rounds looped on the device:
//   active set (generation stamps, ids sorted by rank) -> pair counts c_ij from the key lists of
//   the active instances (each shared key counted from the lower id's list) -> R36 test, lock-free
//   union-find rooted at the min id -> warp per component: T summed in ascending id order, (e, Q)
//   replaced iff strictly higher, obs summed, last_seen max, AABB union, the root's key list sized for
//   the merge -> relabel items (the members' key lists): the root's label inserted (appended to its
//   list when new), the member's tombstoned -> |V|, list lengths, counters, report.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void rf_pair_add(const FrameScratch& X, unsigned long long code, int* err) {
  uint32_t h = (uint32_t)mix64(code) & (uint32_t)(X.RPC - 1);
  for (int probe = 0; probe < X.RPC; ++probe) {
    unsigned long long k = __ldcg(&X.rf_pkey[h]);
    if (k == KEY_EMPTY) {
      k = atomicCAS(&X.rf_pkey[h], KEY_EMPTY, code);
      if (k == KEY_EMPTY) k = code;
    }
    if (k == code) {
      atomicAdd(&X.rf_pcnt[h], 1u);
      return;
    }
    h = (h + 1) & (uint32_t)(X.RPC - 1);
  }
  raise_err(err, DERR_TRIPLES);
}

__device__ uint32_t rf_find(int32_t* par, uint32_t x) {
  while (true) {
    const uint32_t p = (uint32_t)__ldcg(&par[x]);
    if (p == x) return x;
    const uint32_t gp = (uint32_t)__ldcg(&par[p]);
    if (gp != p) atomicCAS(&par[x], (int32_t)p, (int32_t)gp);
    x = p;
  }
}

__global__ void __launch_bounds__(K6_THREADS, 1) k_refine(int f, int S, WinBufs wb, MapState M, FrameScratch X, Params P) {
  const uint32_t G = gridDim.x;
  uint32_t ep = 0;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t gt = blockIdx.x * blockDim.x + tid, gn = G * blockDim.x;
  const uint32_t gw = gt >> 5, gwn = gn >> 5;
  const int Dt = P.Dt, Df = P.Df;
  __shared__ uint32_t gen_s;
  // ---- active set: frame targets and the triples' (still alive) instances, deduplicated ----
  if (tid == 0) gen_s = (uint32_t)(__ldcg((const unsigned long long*)&M.counters[3]) + 1);
  __syncthreads();
  const uint32_t gen = gen_s;
  const uint32_t ntr = min(__ldcg(X.ntrip_last), (uint32_t)X.TCAP);
  const int ntg = *X.ntgt;
  for (uint32_t i = gt; i < ntr + (uint32_t)ntg; i += gn) {
    const uint32_t j = i < ntr ? X.trip_j[i] : X.tgt_root[i - ntr];
    if (!M.alive[j]) continue;
    if (atomicExch(&M.stamp[j], gen) != gen) {
      const uint32_t a = atomicAdd(&X.rf_n[5], 1u);
      if (a < (uint32_t)X.RCAP) X.rf_act[a] = j;
      else raise_err(M.err, DERR_TRIPLES);
    }
  }
  grid_sync(wb.s2bar, G * ++ep);
  if (gt == 0) M.counters[3] = gen;   // (the next frame's association takes gen + 1)
  disc_frame_report& R = X.rep[f];
  for (int round = 0;; ++round) {
    // active ids ascending (rank sort: a few hundred at most), union-find reset, counters reset
    const uint32_t nact = min(__ldcg(&X.rf_n[5]), (uint32_t)X.RCAP);
    for (uint32_t a = gt; a < nact; a += gn) {
      const uint32_t v = __ldcg(&X.rf_act[a]);
      uint32_t rk = 0;
      for (uint32_t b = 0; b < nact; ++b) rk += __ldcg(&X.rf_act[b]) < v;
      X.rf_act2[rk] = v;
      M.local[v] = (int32_t)v;   // union-find parent
    }
    if (gt == 0) { X.rf_n[1] = 0; X.rf_n[2] = 0; X.rf_n[3] = 0; }
    grid_sync(wb.s2bar, G * ++ep);
    // pair counts over the active instances' key lists: key k of V_i with an active label j > i
    for (uint32_t a = blockIdx.x; a < nact; a += G) {
      const uint32_t i = __ldcg(&X.rf_act2[a]);
      const uint32_t Li = M.phys_of[i];
      const unsigned long long off = M.lst_off[Li];
      const uint32_t len = M.lst_len[Li];
      for (uint32_t k = tid; k < len; k += blockDim.x) {
        const uint32_t slot = M.arena[off + k];
        const uint32_t* labs = M.slots[slot].lab;
        int nl = INLINE_LABELS;
        uint32_t nx = M.slots[slot].ovf;
        bool done = false;
        while (!done) {
          for (int c = 0; c < nl; ++c) {
            const uint32_t L = __ldcg(&labs[c]);
            if (L == U32_EMPTY) { done = true; break; }
            if (L == LAB_TOMB || L == Li) continue;
            const uint32_t j = M.id_of[L];
            if (j > i && __ldcg(&M.stamp[j]) == gen && M.alive[j]) rf_pair_add(X, ((unsigned long long)i << 32) | j, M.err);
          }
          if (done || nx == U32_EMPTY) break;
          labs = M.ovf[nx].lab;
          nl = CHUNK_LABELS;
          nx = __ldcg(&M.ovf[nx].next);
        }
      }
    }
    grid_sync(wb.s2bar, G * ++ep);
    // R36 test (warp per pair-table slot), union at the min id; the table is emptied
    for (uint32_t e = gw; e < (uint32_t)X.RPC; e += gwn) {
      const unsigned long long code = __ldcg(&X.rf_pkey[e]);
      if (code == KEY_EMPTY) continue;
      const uint32_t c = __ldcg(&X.rf_pcnt[e]);
      const uint32_t i = (uint32_t)(code >> 32), j = (uint32_t)code;
      const int64_t mn = min(M.vcount[i], M.vcount[j]);
      bool ok = c >= 1 && (double)c >= (double)P.tau_geo * (double)mn;
      if (ok && Dt > 0) {
        const double ti = M.TT[i], tj = M.TT[j];
        const double d = dot_pin_reg(M.T + (size_t)i * Dt, M.T + (size_t)j * Dt, Dt);
        double cosv = -2.0;
        if (ti > 0.0 && tj > 0.0) cosv = __ddiv_rn(__ddiv_rn(d, __dsqrt_rn(ti)), __dsqrt_rn(tj));
        ok = cosv >= (double)P.tau_vis;
      }
      if (lane == 0) {
        if (ok) {
          atomicAdd(&X.rf_n[1], 1u);
          uint32_t a = i, b = j;
          while (true) {
            a = rf_find(M.local, a);
            b = rf_find(M.local, b);
            if (a == b) break;
            if (a > b) { const uint32_t t = a; a = b; b = t; }
            if (atomicCAS(&M.local[b], (int32_t)b, (int32_t)a) == (int32_t)b) break;
          }
        }
        X.rf_pkey[e] = KEY_EMPTY;
        X.rf_pcnt[e] = 0;
      }
      __syncwarp();
    }
    grid_sync(wb.s2bar, G * ++ep);
    if (__ldcg(&X.rf_n[1]) == 0) break;   // fixpoint (uniform)
    // warp per component root (ascending member order = the sorted active list)
    for (uint32_t a = gw; a < nact; a += gwn) {
      const uint32_t r = __ldcg(&X.rf_act2[a]);
      if (rf_find(M.local, r) != r) continue;   // a member, not a root
      uint32_t nm = 0;
      for (uint32_t b = lane; b < nact; b += 32) nm += (X.rf_act2[b] != r && rf_find(M.local, X.rf_act2[b]) == r);
#pragma unroll
      for (int o = 16; o; o >>= 1) nm += __shfl_xor_sync(0xffffffffu, nm, o);
      if (nm == 0) continue;
      // T: ((T_r + T_m1) + T_m2) ..., members ascending
      for (int d = lane; d < Dt; d += 32) {
        double acc = M.T[(size_t)r * Dt + d];
        for (uint32_t b = 0; b < nact; ++b) {
          const uint32_t m = X.rf_act2[b];
          if (m != r && rf_find(M.local, m) == r) acc = __dadd_rn(acc, M.T[(size_t)m * Dt + d]);
        }
        M.T[(size_t)r * Dt + d] = acc;
      }
      __syncwarp();
      if (Dt > 0) {
        const double tt = dot_pin_reg(M.T + (size_t)r * Dt, M.T + (size_t)r * Dt, Dt);
        if (lane == 0) M.TT[r] = tt;
      }
      // (e, Q), obs, last_seen, AABB, key-list capacity, relabel segments (lane 0, ascending)
      uint32_t src = r, base_w = 0;
      unsigned long long off_w = 0, noff_w = 0;
      if (lane == 0) {
        float q = M.q[r];
        int obs = M.obs[r];
        int64_t ls = M.last_seen[r];
        int32_t ab[6];
        for (int k = 0; k < 6; ++k) ab[k] = M.aabb[(size_t)r * 6 + k];
        const uint32_t Lr = M.phys_of[r];
        const uint32_t base = M.lst_len[Lr], cap = M.lst_cap[Lr];
        const unsigned long long off = M.lst_off[Lr];
        uint64_t need = base;
        unsigned long long rel = 0;
        const uint32_t c = atomicAdd(&X.rf_n[2], 1u);
        for (uint32_t b = 0; b < nact; ++b) {
          const uint32_t m = X.rf_act2[b];
          if (m == r || rf_find(M.local, m) != r) continue;
          if (M.q[m] > q) { q = M.q[m]; src = m; }
          obs += M.obs[m];
          ls = max(ls, M.last_seen[m]);
          for (int k = 0; k < 3; ++k) {
            ab[k] = min(ab[k], M.aabb[(size_t)m * 6 + k]);
            ab[3 + k] = max(ab[3 + k], M.aabb[(size_t)m * 6 + 3 + k]);
          }
          const uint32_t Lm = M.phys_of[m];
          const uint32_t sg = atomicAdd(&X.rf_n[3], 1u);
          if (sg < (uint32_t)X.RCAP) {
            X.rf_sL[sg] = Lm;
            X.rf_sc[sg] = c;
            X.rf_sbase[sg] = M.lst_off[Lm];
            X.rf_slen[sg] = M.lst_len[Lm];
          } else {
            raise_err(M.err, DERR_TRIPLES);
          }
          need += M.lst_len[Lm];
          rel += (unsigned long long)M.vcount[m];
          M.lst_len[Lm] = 0;
          M.lst_cap[Lm] = 0;
          M.alive[m] = 0;
          M.phys_of[m] = U32_EMPTY;
        }
        unsigned long long noff = off;
        if (need > cap) {   // the root's list moves to a region sized for the merge (old entries copied below)
          const uint32_t nc = (uint32_t)max(max(2ull * cap, (unsigned long long)need), 64ull);
          const unsigned long long o = atomicAdd(M.arena_top, (unsigned long long)nc);
          if (o + nc > M.ARENA) {
            raise_err(M.err, DERR_ARENA);
          } else {
            noff = o;
            M.lst_off[Lr] = o;
            M.lst_cap[Lr] = nc;
          }
        }
        X.rf_croot[c] = r;
        X.rf_cbase[c] = base;
        X.rf_coff[c] = noff;
        X.rf_cadd[c] = 0;
        M.q[r] = q;
        M.obs[r] = obs;
        M.last_seen[r] = ls;
        for (int k = 0; k < 6; ++k) M.aabb[(size_t)r * 6 + k] = ab[k];
        atomicAdd((unsigned long long*)&R.merged_away, (unsigned long long)nm);
        atomicAdd((unsigned long long*)&R.refine_merged, (unsigned long long)nm);
        atomicAdd((unsigned long long*)&R.relabeled, rel);
        base_w = base;
        off_w = off;
        noff_w = noff;
      }
      src = __shfl_sync(0xffffffffu, src, 0);
      base_w = __shfl_sync(0xffffffffu, base_w, 0);
      off_w = __shfl_sync(0xffffffffu, off_w, 0);
      noff_w = __shfl_sync(0xffffffffu, noff_w, 0);
      if (noff_w != off_w)   // the moved list's old entries, copied by the warp
        for (uint32_t k = lane; k < base_w; k += 32) M.arena[noff_w + k] = M.arena[off_w + k];
      if (src != r)
        for (int d = lane; d < Df; d += 32) M.E[(size_t)r * Df + d] = M.E[(size_t)src * Df + d];
    }
    grid_sync(wb.s2bar, G * ++ep);
    // relabel segment prefix (a few hundred segments: one thread)
    const uint32_t nseg = min(__ldcg(&X.rf_n[3]), (uint32_t)X.RCAP);
    if (gt == 0) {
      uint32_t acc = 0;
      for (uint32_t g = 0; g < nseg; ++g) { X.rf_spre[g] = acc; acc += X.rf_slen[g]; }
      X.rf_spre[nseg] = acc;
    }
    grid_sync(wb.s2bar, G * ++ep);
    // relabel items: the root's label onto each member key (appended to the root's list when new),
    // the member's label tombstoned
    const uint32_t nit = __ldcg(&X.rf_spre[nseg]);
    int delta = 0;
    for (uint32_t it = gt; it < nit; it += gn) {
      int lo = 0, hi = (int)nseg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldcg(&X.rf_spre[mid]) <= it) lo = mid;
        else hi = mid - 1;
      }
      const uint32_t c = X.rf_sc[lo];
      const uint32_t slot = M.arena[X.rf_sbase[lo] + (it - X.rf_spre[lo])];
      const uint32_t Lr = M.phys_of[X.rf_croot[c]];
      if (label_insert(M, slot, Lr)) {
        const uint32_t pos = atomicAdd(&X.rf_cadd[c], 1u);
        M.arena[X.rf_coff[c] + X.rf_cbase[c] + pos] = slot;
        ++delta;
      }
      if (label_tomb(M, slot, X.rf_sL[lo])) --delta;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) delta += __shfl_xor_sync(0xffffffffu, delta, o);
    if (lane == 0 && delta) atomicAdd((unsigned long long*)&M.counters[2], (unsigned long long)(int64_t)delta);
    grid_sync(wb.s2bar, G * ++ep);
    // tails: the roots' |V| and list lengths; the active set keeps the survivors
    const uint32_t ncomp = min(__ldcg(&X.rf_n[2]), (uint32_t)X.RCAP);
    for (uint32_t c = gt; c < ncomp; c += gn) {
      const uint32_t r = X.rf_croot[c];
      const uint32_t add = X.rf_cadd[c];
      M.lst_len[M.phys_of[r]] = X.rf_cbase[c] + add;
      M.vcount[r] += add;
    }
    for (int s = (int)gt; s < S; s += (int)gn) {   // the detections' instances follow the merges (debug export)
      const int64_t t = X.det_id[s];
      if (t >= 0 && !M.alive[t]) X.det_id[s] = rf_find(M.local, (uint32_t)t);
    }
    if (gt == 0) {
      R.refine_rounds += 1;
      uint32_t w = 0;
      for (uint32_t a = 0; a < nact; ++a)
        if (M.alive[X.rf_act2[a]]) X.rf_act[w++] = X.rf_act2[a];
      X.rf_n[5] = w;
      M.counters[1] -= (int64_t)(nact - w);
    }
    grid_sync(wb.s2bar, G * ++ep);
  }
  if (gt == 0) {   // the report's live counts after the refinement
    R.live_instances = M.counters[1];
    R.live_memberships = M.counters[2];
    R.new_memberships = M.counters[2] - *X.live_before;
    X.rf_n[5] = 0;
  }
}

void launch_refine(int f, int S, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P, int grid,
                   cudaStream_t st) {
  cudaMemsetAsync(wb.s2bar, 0, sizeof(uint32_t), st);
  int ff = f, SS = S;
  void* args[] = {(void*)&ff, (void*)&SS, (void*)&wb, (void*)&M, (void*)&X, (void*)&P};
  cudaLaunchCooperativeKernel((const void*)k_refine, dim3(grid), dim3(K6_THREADS), args, 0, st);
  debug_check(st, "k_refine", f);
}

int launch_stage2(const WinDesc& wd, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P,
                  bool sem, int nsm, int nres, uint32_t* tag_seq, int spec_mode, cudaStream_t st) {
  const size_t sm6 = k6_smem_bytes(wb.SMAX, X.TCS);
  static size_t set_for = 0;
  if (set_for != sm6) {
    cudaFuncSetAttribute(k_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
    set_for = sm6;
  }
  const int grid = nres > 0 ? nres : std::min(16, nsm);
  static const int prof = getenv("DISC_S2PROF") ? atoi(getenv("DISC_S2PROF")) : 0;
  // cooperative launch: its CTAs wait on one another at the grid barriers, so co-residency must
  // be guaranteed, not assumed
  int semi = sem ? 1 : 0;
  // speculative work during the association (k_stage2): 2 counting + corrections, 1 slots, 0 hints
  int spec = spec_mode;
  int f0 = 0, fn = wd.n;
  // slot-chain tags of the speculatively counted frames: the map's own sequence (never reused
  // between clears of M.slh, so no clearing per frame); 0 = none
  if (*tag_seq == 0 || *tag_seq + (uint32_t)wd.n + 1 < *tag_seq) {   // first use / wrap: clear, restart
    cudaMemsetAsync(M.slh, 0, sizeof(unsigned long long) * M.MC, st);
    *tag_seq = 1;
  }
  uint32_t tag0 = *tag_seq;
  *tag_seq += (uint32_t)wd.n + 1;
  void* args[] = {(void*)&wd, (void*)&wb, (void*)&M, (void*)&X, (void*)&P, (void*)&semi, (void*)&prof, (void*)&spec,
                  (void*)&f0, (void*)&fn, (void*)&tag0};
  if (!P.refine) {
    cudaLaunchCooperativeKernel((const void*)k_stage2, dim3(grid), dim3(K6_THREADS), args, sm6, st);
    debug_check(st, "k_stage2", -1);
    return 1;
  }
  // refine_active: each frame's update, then its refinement, before the next frame's lookup
  for (int f = 0; f < wd.n; ++f) {
    f0 = f;
    fn = 1;
    cudaMemsetAsync(wb.s2bar, 0, sizeof(uint32_t), st);
    cudaLaunchCooperativeKernel((const void*)k_stage2, dim3(grid), dim3(K6_THREADS), args, sm6, st);
    debug_check(st, "k_stage2", f);
    launch_refine(f, wd.f[f].S, wb, M, X, P, grid, st);
  }
  return 2 * wd.n;
}

}  // namespace disc
