// k_frame.cu -- stage 1 of the DISC hot path: per-frame-independent work, batched over a
// window of frames.
//
//  K0  k_win_init      reset the window's per-mask accumulators
//  K1  k_mask_pass     depth -> pinned fp32 world point -> voxel key (R5) -> frame key table;
//                      every mask byte read once (16-B streaming loads): area, bbox, per-patch
//                      pixel counts, unique (s, key) pairs (|V_s|), pixel normal sums (R21)
//  K2  k_pairs         pair records for stage 2, detection AABBs, S_angle terms (Eq.3)
//  K3  k_fbar_part / k_fbar / k_resid   distinctiveness map inputs (Eq.1)
//  K4  k_detect        mask filter (A1), D-weighted pooling, Q (Eq.2-3) and the
//                      tracking feature t_s (R15)
#include "disc_common.cuh"
#include "disc_launch.h"

namespace disc {

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------

// R5: p_w = R (d K^-1 [u,v,1]) + t, pinned fp32 order, no contraction.
// xa = (float)u - cx, divided by fx (exact IEEE ops; precomputed per column / row).
__device__ __forceinline__ void world_point(const FrameDesc& F, float xa, float yb, float d, float p[3]) {
  const float xc = __fmul_rn(xa, d);
  const float yc = __fmul_rn(yb, d);
  const float zc = d;
  p[0] = __fmaf_rn(F.pose[0], xc, __fmaf_rn(F.pose[1], yc, __fmaf_rn(F.pose[2], zc, F.pose[3])));
  p[1] = __fmaf_rn(F.pose[4], xc, __fmaf_rn(F.pose[5], yc, __fmaf_rn(F.pose[6], zc, F.pose[7])));
  p[2] = __fmaf_rn(F.pose[8], xc, __fmaf_rn(F.pose[9], yc, __fmaf_rn(F.pose[10], zc, F.pose[11])));
}

__device__ __forceinline__ bool depth_valid(float d, const Params& P) {
  return isfinite(d) && d > P.dmin && d < P.dmax;
}

// R5/R6: key = floor(p / r) per component, division (not multiplication by 1/r)
__device__ __forceinline__ bool point_key(const float p[3], float r, uint64_t& key) {
  int k[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float q = floorf(__fdiv_rn(p[i], r));
    if (!(q >= -1048576.0f && q < 1048576.0f)) return false;
    k[i] = (int)q;
  }
  key = pack_key(k[0], k[1], k[2]);
  return true;
}

__device__ __forceinline__ uint32_t ktab_insert(unsigned long long* tab, uint32_t mask, uint64_t key,
                                                int* err) {
  uint32_t h = (uint32_t)mix64(key) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    unsigned long long cur = __ldcg(&tab[h]);
    if (cur == key) return h;
    if (cur == KEY_EMPTY) {
      const unsigned long long old = atomicCAS(&tab[h], KEY_EMPTY, (unsigned long long)key);
      if (old == KEY_EMPTY || old == key) return h;
    }
    h = (h + 1) & mask;
  }
  raise_err(err, DERR_FRAME_PAIRS);
  return U32_EMPTY;
}

// returns slot; *fresh = true iff this call inserted the code
__device__ __forceinline__ uint32_t ptab_insert(uint32_t* tab, uint32_t mask, uint32_t code, bool* fresh,
                                                int* err) {
  uint32_t h = mix32(code) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    const uint32_t cur = __ldcg(&tab[h]);
    if (cur == code) { *fresh = false; return h; }
    if (cur == U32_EMPTY) {
      const uint32_t old = atomicCAS(&tab[h], U32_EMPTY, code);
      if (old == U32_EMPTY) { *fresh = true; return h; }
      if (old == code) { *fresh = false; return h; }
    }
    h = (h + 1) & mask;
  }
  raise_err(err, DERR_FRAME_PAIRS);
  *fresh = false;
  return U32_EMPTY;
}

__device__ __forceinline__ uint4 ld_stream16(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------------------------------------
// K0
// ------------------------------------------------------------------------------------------
__global__ void k_win_init(WinDesc wd, WinBufs wb) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const int S = wd.f[f].S;
  for (int s = threadIdx.x + blockIdx.x * blockDim.x; s < S; s += blockDim.x * gridDim.x) {
    const size_t i = (size_t)f * wb.SMAX + s;
    wb.area[i] = 0;
    wb.vs[i] = 0;
    wb.ang_sum[i] = 0.f;
    wb.ang_cnt[i] = 0;
    wb.bbox[4 * i + 0] = INT32_MAX;
    wb.bbox[4 * i + 1] = INT32_MAX;
    wb.bbox[4 * i + 2] = -1;
    wb.bbox[4 * i + 3] = -1;
    for (int k = 0; k < 3; ++k) {
      wb.daabb[6 * i + k] = INT32_MAX;
      wb.daabb[6 * i + 3 + k] = INT32_MIN;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wb.npairs[f] = 0;
    wb.oor[f] = 0;
  }
}

// ------------------------------------------------------------------------------------------
// K1: one CTA per (patch row, frame).  The CTA's pixels are the image rows that map to patch
// row `band` (R17 floor mapping), so it owns cnt[s][band][*] outright (no global atomics
// for per-patch counts).  A thread handles 16 consecutive pixels: keys once, then one
// 16-byte streaming load per mask plane.
// ------------------------------------------------------------------------------------------
constexpr int K1_THREADS = 256;
constexpr int K1_PLIST = 2048;

template <bool SEM>
__global__ void __launch_bounds__(K1_THREADS) k_mask_pass(WinDesc wd, WinBufs wb, Params P, int* err, int rows_cap) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int band = blockIdx.x;
  if (band >= F.Hp) return;
  const int H = F.H, W = F.W, S = F.S, Hp = F.Hp, Wp = F.Wp;
  const int64_t HW = (int64_t)H * W;
  const int v0 = (int)(((int64_t)band * H + Hp - 1) / Hp);
  const int v1 = (int)(((int64_t)(band + 1) * H + Hp - 1) / Hp);
  const int64_t i0 = (int64_t)v0 * W, i1 = (int64_t)v1 * W;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* cnt_s = (uint32_t*)smem_raw;                       // [S][Wp]
  int32_t* bb_s = (int32_t*)(cnt_s + (size_t)S * Wp);         // [S][4]
  uint32_t* vs_s = (uint32_t*)(bb_s + 4 * S);                  // [S]
  uint32_t* pl_s = vs_s + S;                                   // [K1_PLIST]
  float* xa_s = (float*)(pl_s + K1_PLIST);                     // [W]  ((float)u - cx) / fx
  uint16_t* pc_s = (uint16_t*)(xa_s + W);                      // [W]  patch column of u
  float* yb_s = (float*)(pc_s + ((W + 1) & ~1));               // rows v0-1 .. v1: ((float)v - cy)/fy
  unsigned long long* ks_all = (unsigned long long*)(((uintptr_t)(yb_s + rows_cap) + 15) & ~(uintptr_t)15);
  unsigned long long* ks = ks_all + threadIdx.x;               // ks[j * K1_THREADS]: packed key
  __shared__ uint32_t npl_s, oor_s;

  for (int i = threadIdx.x; i < S * Wp; i += blockDim.x) cnt_s[i] = 0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    bb_s[4 * i + 0] = INT32_MAX; bb_s[4 * i + 1] = INT32_MAX;
    bb_s[4 * i + 2] = -1; bb_s[4 * i + 3] = -1;
    vs_s[i] = 0;
  }
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    xa_s[u] = __fdiv_rn(__fsub_rn((float)u, F.cx), F.fx);
    pc_s[u] = (uint16_t)(((int64_t)u * Wp) / W);
  }
  for (int v = v0 - 1 + (int)threadIdx.x; v <= v1; v += blockDim.x)
    yb_s[v - (v0 - 1)] = __fdiv_rn(__fsub_rn((float)v, F.cy), F.fy);
  if (threadIdx.x == 0) { npl_s = 0; oor_s = 0; }
  __syncthreads();

  const uint32_t tmask = (uint32_t)wb.PC - 1;
  unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
  float* nsum = wb.nsum + (size_t)f * wb.PC * 3;
  const float r = P.r;

  auto ybv = [&](int v) { return yb_s[v - (v0 - 1)]; };
  // world point of an arbitrary pixel (normals need neighbours outside the band)
  auto wp_at = [&](int u, int v, float p[3]) -> bool {
    const float d = F.depth[(int64_t)v * W + u];
    if (!depth_valid(d, P)) return false;
    world_point(F, xa_s[u], (v >= v0 - 1 && v <= v1) ? ybv(v) : __fdiv_rn(__fsub_rn((float)v, F.cy), F.fy), d, p);
    return true;
  };
  // R21 pixel normal (fp32): (P(u+1,v)-P(u-1,v)) x (P(u,v+1)-P(u,v-1)), oriented to the camera
  auto pixel_normal = [&](int u, int v, const float pc[3], float n[3]) -> bool {
    if (u < 1 || u + 1 >= W || v < 1 || v + 1 >= H) return false;
    float pl[3], pr[3], pu[3], pd[3];
    if (!wp_at(u - 1, v, pl) || !wp_at(u + 1, v, pr) || !wp_at(u, v - 1, pu) || !wp_at(u, v + 1, pd)) return false;
    const float a0 = pr[0] - pl[0], a1 = pr[1] - pl[1], a2 = pr[2] - pl[2];
    const float b0 = pd[0] - pu[0], b1 = pd[1] - pu[1], b2 = pd[2] - pu[2];
    n[0] = a1 * b2 - a2 * b1;
    n[1] = a2 * b0 - a0 * b2;
    n[2] = a0 * b1 - a1 * b0;
    if (n[0] == 0.f && n[1] == 0.f && n[2] == 0.f) return false;
    const float o = n[0] * (F.pose[3] - pc[0]) + n[1] * (F.pose[7] - pc[1]) + n[2] * (F.pose[11] - pc[2]);
    if (o < 0.f) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
    return true;
  };

  const int64_t c0 = i0 >> 4, c1 = (i1 + 15) >> 4;
  uint32_t my_oor = 0;
  for (int64_t ch = c0 + threadIdx.x; ch < c1; ch += blockDim.x) {
    const int64_t ib = ch << 4;
    int u_start = (int)(ib % W), v_start = (int)(ib / W);
    // ---- pixel pass: keys of the 16 pixels ----
    uint32_t okbits = 0, inband = 0;
    {
      int u = u_start, v = v_start;
      for (int j = 0; j < 16; ++j) {
        const int64_t i = ib + j;
        if (i >= i0 && i < i1) {
          inband |= 1u << j;
          const float d = F.depth[i];
          if (depth_valid(d, P)) {
            float p[3];
            world_point(F, xa_s[u], ybv(v), d, p);
            uint64_t key;
            if (point_key(p, r, key)) {
              ks[j * K1_THREADS] = key;
              okbits |= 1u << j;
            } else {
              my_oor++;
            }
          }
        }
        if (++u == W) { u = 0; ++v; }
      }
    }
    if (!inband) continue;
    // ---- mask pass ----
    for (int s = 0; s < S; ++s) {
      uint32_t w[4];
      if (F.vec16) {
        const uint4 m = ld_stream16(F.masks + (size_t)s * HW + ib);
        w[0] = m.x; w[1] = m.y; w[2] = m.z; w[3] = m.w;
      } else {
        for (int q = 0; q < 4; ++q) {
          uint32_t x = 0;
          for (int b = 0; b < 4; ++b) {
            const int64_t i = ib + 4 * q + b;
            if (i < HW) x |= (uint32_t)(F.masks[(size_t)s * HW + i] != 0) << (8 * b);
          }
          w[q] = x;
        }
      }
      if ((w[0] | w[1] | w[2] | w[3]) == 0) continue;
      uint32_t set = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t nz = __vcmpne4(w[q], 0u) & 0x01010101u;
        set |= ((nz & 1u) | ((nz >> 7) & 2u) | ((nz >> 14) & 4u) | ((nz >> 21) & 8u)) << (4 * q);
      }
      set &= inband;
      if (!set) continue;
      // per-patch pixel counts (regardless of depth) and bbox
      int umin = INT32_MAX, umax = -1, vmin = INT32_MAX, vmax = -1;
      {
        int u = u_start, v = v_start;
        int run_pc = -1;
        uint32_t run_n = 0;
        for (int j = 0; j < 16; ++j) {
          if (set & (1u << j)) {
            umin = min(umin, u); umax = max(umax, u);
            vmin = min(vmin, v); vmax = max(vmax, v);
            const int pc = pc_s[u];
            if (pc != run_pc) {
              if (run_n) atomicAdd(&cnt_s[s * Wp + run_pc], run_n);
              run_pc = pc;
              run_n = 0;
            }
            run_n++;
          }
          if (++u == W) { u = 0; ++v; }
        }
        if (run_n) atomicAdd(&cnt_s[s * Wp + run_pc], run_n);
      }
      atomicMin(&bb_s[4 * s + 0], umin);
      atomicMin(&bb_s[4 * s + 1], vmin);
      atomicMax(&bb_s[4 * s + 2], umax);
      atomicMax(&bb_s[4 * s + 3], vmax);
      // unique (s, key) pairs, run-compressed along the chunk
      uint32_t pk = set & okbits;
      if (!pk) continue;
      {
        int u = u_start, v = v_start;
        uint64_t run_key = KEY_EMPTY;
        uint32_t run_pslot = U32_EMPTY;
        float ns0 = 0.f, ns1 = 0.f, ns2 = 0.f;
        bool have_n = false;
        for (int j = 0; j < 16; ++j) {
          if (pk & (1u << j)) {
            const uint64_t kj = ks[j * K1_THREADS];
            if (kj != run_key) {
              if (SEM && have_n && run_pslot != U32_EMPTY) {
                atomicAdd(&nsum[3 * run_pslot + 0], ns0);
                atomicAdd(&nsum[3 * run_pslot + 1], ns1);
                atomicAdd(&nsum[3 * run_pslot + 2], ns2);
              }
              ns0 = ns1 = ns2 = 0.f;
              have_n = false;
              run_key = kj;
              // frame key table: only keys of mask pixels enter it (K5 releases every cell)
              const uint32_t kslot = ktab_insert(ktab, tmask, kj, err);
              bool fresh = false;
              run_pslot = kslot == U32_EMPTY ? U32_EMPTY
                                             : ptab_insert(ptab, tmask, ((uint32_t)s << 24) | kslot, &fresh, err);
              if (fresh) {
                DISC_CHECK(err, __ldcg(&ptab[run_pslot]) == (((uint32_t)s << 24) | kslot));
                DISC_CHECK(err, __ldcg(&ktab[kslot]) == kj);
                atomicAdd(&vs_s[s], 1u);
                const uint32_t li = atomicAdd(&npl_s, 1u);
                if (li < K1_PLIST) {
                  pl_s[li] = run_pslot;
                } else {
                  const uint32_t gi = atomicAdd(&wb.npairs[f], 1u);
                  if (gi < (uint32_t)wb.PMAX) wb.plist[(size_t)f * wb.PMAX + gi] = run_pslot;
                  else raise_err(err, DERR_FRAME_PAIRS);
                }
              }
            }
            if (SEM) {
              float p[3], n[3];
              world_point(F, xa_s[u], ybv(v), F.depth[ib + j], p);
              if (pixel_normal(u, v, p, n)) {
                ns0 += n[0]; ns1 += n[1]; ns2 += n[2];
                have_n = true;
              }
            }
          }
          if (++u == W) { u = 0; ++v; }
        }
        if (SEM && have_n && run_pslot != U32_EMPTY) {
          atomicAdd(&nsum[3 * run_pslot + 0], ns0);
          atomicAdd(&nsum[3 * run_pslot + 1], ns1);
          atomicAdd(&nsum[3 * run_pslot + 2], ns2);
        }
      }
    }
  }
  if (my_oor) atomicAdd(&oor_s, my_oor);
  __syncthreads();

  // ---- flush ----
  uint32_t* cnt_g = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP;
  for (int i = threadIdx.x; i < S * Wp; i += blockDim.x) {
    const int s = i / Wp, pc = i - s * Wp;
    cnt_g[(size_t)s * wb.PMAXP + (size_t)band * Wp + pc] = cnt_s[i];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = warp; s < S; s += blockDim.x >> 5) {
    uint32_t a = 0;
    for (int pc = lane; pc < Wp; pc += 32) a += cnt_s[s * Wp + pc];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0 && a) {
      const size_t gi = (size_t)f * wb.SMAX + s;
      atomicAdd(&wb.area[gi], a);
      atomicMin(&wb.bbox[4 * gi + 0], bb_s[4 * s + 0]);
      atomicMin(&wb.bbox[4 * gi + 1], bb_s[4 * s + 1]);
      atomicMax(&wb.bbox[4 * gi + 2], bb_s[4 * s + 2]);
      atomicMax(&wb.bbox[4 * gi + 3], bb_s[4 * s + 3]);
      if (vs_s[s]) atomicAdd(&wb.vs[gi], vs_s[s]);
    }
  }
  __shared__ uint32_t base_s;
  const uint32_t n = min(npl_s, (uint32_t)K1_PLIST);
  if (threadIdx.x == 0) {
    base_s = n ? atomicAdd(&wb.npairs[f], n) : 0;
    if (oor_s) atomicAdd(&wb.oor[f], (unsigned long long)oor_s);
  }
  __syncthreads();
  if (base_s + n > (uint32_t)wb.PMAX) {
    if (threadIdx.x == 0) raise_err(err, DERR_FRAME_PAIRS);
    return;
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    DISC_CHECK(err, pl_s[i] < (uint32_t)wb.PC && __ldcg(&ptab[pl_s[i]]) != U32_EMPTY);
    wb.plist[(size_t)f * wb.PMAX + base_s + i] = pl_s[i];
  }
}

// ------------------------------------------------------------------------------------------
// K2: pair records (key, s, frame-key slot) for stage 2; detection key-space AABBs;
// S_angle terms max(0, -r_v . n_v) (Eq.3, R21) in semantic mode.  Clears the pair table.
// ------------------------------------------------------------------------------------------
constexpr int K2_THREADS = 256;

template <bool SEM>
__global__ void __launch_bounds__(K2_THREADS) k_pairs(WinDesc wd, WinBufs wb, Params P, int* err) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int S = F.S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* ab_s = (int32_t*)smem_raw;            // [S][6]
  float* as_s = (float*)(ab_s + 6 * S);          // [S]
  uint32_t* ac_s = (uint32_t*)(as_s + S);        // [S]
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    for (int k = 0; k < 3; ++k) { ab_s[6 * s + k] = INT32_MAX; ab_s[6 * s + 3 + k] = INT32_MIN; }
    as_s[s] = 0.f;
    ac_s[s] = 0;
  }
  __syncthreads();
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
  const unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  float* nsum = wb.nsum + (size_t)f * wb.PC * 3;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < np; idx += gridDim.x * blockDim.x) {
    const uint32_t ps = wb.plist[fo + idx];
    if (ps >= (uint32_t)wb.PC) {
      atomicCAS(err, 0, 1000 + __LINE__);
      continue;
    }
    const uint32_t code = ptab[ps];
    const uint32_t s = code >> 24, ks = code & 0xFFFFFFu;
    if (code == U32_EMPTY) {
      atomicCAS(err, 0, 1000 + __LINE__);
      continue;
    }
    if (s >= (uint32_t)S || ks >= (uint32_t)wb.PC) {
      atomicCAS(err, 0, 1000 + __LINE__);
      continue;
    }
    const uint64_t key = ktab[ks];
    wb.pkey[fo + idx] = key;
    wb.pinfo[fo + idx] = s;
    wb.pfk[fo + idx] = ks;
    DISC_CHECK(err, atomicExch(&ptab[ps], U32_EMPTY) == code);
    int k3[3];
    unpack_key(key, k3[0], k3[1], k3[2]);
    for (int a = 0; a < 3; ++a) {
      atomicMin(&ab_s[6 * s + a], k3[a]);
      atomicMax(&ab_s[6 * s + 3 + a], k3[a]);
    }
    if (SEM) {
      const float n0 = nsum[3 * ps], n1 = nsum[3 * ps + 1], n2 = nsum[3 * ps + 2];
      nsum[3 * ps] = 0.f; nsum[3 * ps + 1] = 0.f; nsum[3 * ps + 2] = 0.f;
      const float nl = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
      if (nl > 0.f) {
        const float r0 = ((float)k3[0] + 0.5f) * P.r - F.pose[3];
        const float r1 = ((float)k3[1] + 0.5f) * P.r - F.pose[7];
        const float r2 = ((float)k3[2] + 0.5f) * P.r - F.pose[11];
        const float rl = sqrtf(r0 * r0 + r1 * r1 + r2 * r2);
        if (rl > 0.f) {
          const float dot = (r0 * n0 + r1 * n1 + r2 * n2) / (rl * nl);
          atomicAdd(&as_s[s], fmaxf(0.f, -dot));
          atomicAdd(&ac_s[s], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const size_t gi = (size_t)f * wb.SMAX + s;
    if (ab_s[6 * s] != INT32_MAX) {
      for (int a = 0; a < 3; ++a) {
        atomicMin(&wb.daabb[6 * gi + a], ab_s[6 * s + a]);
        atomicMax(&wb.daabb[6 * gi + 3 + a], ab_s[6 * s + 3 + a]);
      }
    }
    if (SEM && ac_s[s]) {
      atomicAdd(&wb.ang_sum[gi], as_s[s]);
      atomicAdd(&wb.ang_cnt[gi], ac_s[s]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// K3: Eq.1 inputs.  fbar = mean_p f_p (fp64 partial sums, fixed-order reduction) and
// r_p = |f_p - fbar| (fp32, one warp per patch).  rbar and D_p = r_p / (rbar + eps) are
// formed in K4 (fixed-order reduction, per detection CTA).
// ------------------------------------------------------------------------------------------
constexpr int K3_ROWS = 64;

__global__ void __launch_bounds__(256) k_fbar_part(WinDesc wd, WinBufs wb, int Df) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  if (!F.feats) return;
  const int P = F.Hp * F.Wp;
  const int ch = blockIdx.x;
  const int p0 = ch * K3_ROWS;
  if (p0 >= P) return;
  const int p1 = min(P, p0 + K3_ROWS);
  double* part = wb.fpart + ((size_t)f * wb.FCHUNKS + ch) * Df;
  for (int d4 = threadIdx.x; d4 < Df / 4; d4 += blockDim.x) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int p = p0; p < p1; ++p) {
      const float4 x = __ldg((const float4*)(F.feats + (size_t)p * Df) + d4);
      a0 += x.x; a1 += x.y; a2 += x.z; a3 += x.w;
    }
    part[4 * d4 + 0] = a0; part[4 * d4 + 1] = a1; part[4 * d4 + 2] = a2; part[4 * d4 + 3] = a3;
  }
}

__global__ void __launch_bounds__(256) k_fbar(WinDesc wd, WinBufs wb, int Df) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  if (!F.feats) return;
  const int P = F.Hp * F.Wp;
  const int nch = (P + K3_ROWS - 1) / K3_ROWS;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < Df; d += gridDim.x * blockDim.x) {
    double a = 0;
    for (int c = 0; c < nch; ++c) a += wb.fpart[((size_t)f * wb.FCHUNKS + c) * Df + d];
    wb.fbar[(size_t)f * Df + d] = (float)(a / (double)P);
  }
}

__global__ void __launch_bounds__(256) k_resid(WinDesc wd, WinBufs wb, int Df) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  if (!F.feats) return;
  const int P = F.Hp * F.Wp;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const float4* fb = (const float4*)(wb.fbar + (size_t)f * Df);
  for (int p = warp; p < P; p += nw) {
    const float4* row = (const float4*)(F.feats + (size_t)p * Df);
    float acc = 0.f;
    for (int d4 = lane; d4 < Df / 4; d4 += 32) {
      const float4 x = __ldg(row + d4);
      const float4 m = fb[d4];
      const float a = x.x - m.x, b = x.y - m.y, c = x.z - m.z, e = x.w - m.w;
      acc = fmaf(a, a, acc); acc = fmaf(b, b, acc); acc = fmaf(c, c, acc); acc = fmaf(e, e, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) wb.rp[(size_t)f * wb.PMAXP + p] = sqrtf(acc);
  }
}

// ------------------------------------------------------------------------------------------
// K4: one CTA per (mask, frame).
// ------------------------------------------------------------------------------------------
constexpr int K4_THREADS = 256;

__device__ __forceinline__ double block_sum_d(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// R15 pinned fp64 dot over a warp: lane l accumulates d = l, l+32, ... ascending with fma,
// then the xor butterfly 16, 8, 4, 2, 1.
__device__ __forceinline__ double dot_pin_warp(const double* a, const double* b, int n) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int d = lane; d < n; d += 32) acc = __fma_rn(a[d], b[d], acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  return acc;
}

template <bool SEM>
__global__ void __launch_bounds__(K4_THREADS) k_detect(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int s = blockIdx.x;
  if (s >= F.S) return;
  const int H = F.H, W = F.W, Hp = F.Hp, Wp = F.Wp, Df = P.Df, Dt = P.Dt;
  const size_t gi = (size_t)f * wb.SMAX + s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* red = (double*)smem_raw;                 // [33]
  double* u_s = red + 40;                          // [Dt]

  // ---- A1: mask filter (R8), first failing reason wins: area==0, conf, aspect, area ----
  const uint32_t area = wb.area[gi];
  const int umin = wb.bbox[4 * gi + 0], vmin = wb.bbox[4 * gi + 1];
  const int umax = wb.bbox[4 * gi + 2], vmax = wb.bbox[4 * gi + 3];
  const float conf = F.conf ? F.conf[s] : 1.0f;
  int status = 0;
  if (area == 0) status = 1;
  else if (conf < P.min_conf) status = 2;
  else {
    const int64_t bw = umax - umin + 1, bh = vmax - vmin + 1;
    const int64_t lo = min(bw, bh), hi = max(bw, bh);
    if ((double)hi > (double)P.max_aspect * (double)lo) status = 3;
    else if ((int64_t)area < (int64_t)P.min_area) status = 1;
    else if (wb.vs[gi] == 0) status = 4;            // O3 no valid depth
  }
  float* qf = wb.qf + 6 * gi;
  if (status != 0) {
    if (threadIdx.x == 0) {
      wb.status[gi] = status;
      for (int k = 0; k < 6; ++k) qf[k] = k == 4 ? -1.f : 0.f;
      wb.tok[gi] = 0;
    }
    return;
  }
  const int pr0 = (int)((int64_t)vmin * Hp / H), pr1 = (int)((int64_t)vmax * Hp / H);
  const int pc0 = (int)((int64_t)umin * Wp / W), pc1 = (int)((int64_t)umax * Wp / W);
  const uint32_t* cnt = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP + (size_t)s * wb.PMAXP;
  auto rows_of = [&](int i) { return (int)(((int64_t)(i + 1) * H + Hp - 1) / Hp - ((int64_t)i * H + Hp - 1) / Hp); };
  auto cols_of = [&](int j) { return (int)(((int64_t)(j + 1) * W + Wp - 1) / Wp - ((int64_t)j * W + Wp - 1) / Wp); };

  if (SEM && F.feats) {
    // rbar: fixed-order reduction of r_p over all P patches (Eq.1 denominator)
    const int Pn = Hp * Wp;
    const float* rp = wb.rp + (size_t)f * wb.PMAXP;
    double a = 0;
    for (int p = threadIdx.x; p < Pn; p += blockDim.x) a += (double)rp[p];
    const double rbar = block_sum_d(a, red) / (double)Pn;
    const double inv = 1.0 / (rbar + (double)P.eps);
    // weights: w = D cnt/npix if cnt >= cover_min npix (exact), pass 1 = sums
    double wsum = 0, dnum = 0, dden = 0;
    const int npr = pr1 - pr0 + 1, npc = pc1 - pc0 + 1;
    for (int k = threadIdx.x; k < npr * npc; k += blockDim.x) {
      const int i = pr0 + k / npc, j = pc0 + k % npc;
      const uint32_t c = cnt[i * Wp + j];
      if (!c) continue;
      const double npix = (double)rows_of(i) * (double)cols_of(j);
      const double D = (double)rp[i * Wp + j] * inv;
      const double cov = (double)c / npix;
      dnum += cov * D;
      dden += cov;
      if ((double)c >= (double)P.cover_min * npix) wsum += D * cov;
    }
    wsum = block_sum_d(wsum, red);
    dnum = block_sum_d(dnum, red);
    dden = block_sum_d(dden, red);
    const bool fallback = !(wsum > 0.0);
    const double dbar = dden > 0 ? dnum / dden : 0.0;
    // pooling y = sum_p w_p f_p, ascending p; each thread owns 4 columns per step
    float* emb = wb.emb + gi * Df;
    double yy = 0;
    for (int d4 = threadIdx.x; d4 < Df / 4; d4 += blockDim.x) {
      float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = pr0; i <= pr1; ++i)
        for (int j = pc0; j <= pc1; ++j) {
          const uint32_t c = cnt[i * Wp + j];
          if (!c) continue;
          float w;
          if (fallback) {
            w = 1.0f;
          } else {
            const double npix = (double)rows_of(i) * (double)cols_of(j);
            if (!((double)c >= (double)P.cover_min * npix)) continue;
            w = (float)((double)rp[i * Wp + j] * inv * ((double)c / npix));
          }
          const float4 x = __ldg((const float4*)(F.feats + ((size_t)i * Wp + j) * Df) + d4);
          y.x = fmaf(w, x.x, y.x); y.y = fmaf(w, x.y, y.y); y.z = fmaf(w, x.z, y.z); y.w = fmaf(w, x.w, y.w);
        }
      ((float4*)emb)[d4] = y;
      yy += (double)y.x * y.x + (double)y.y * y.y + (double)y.z * y.z + (double)y.w * y.w;
    }
    yy = block_sum_d(yy, red);
    if (!(yy > 0.0)) {
      if (threadIdx.x == 0) {
        wb.status[gi] = 5;   // nofeat
        for (int k = 0; k < 6; ++k) qf[k] = k == 4 ? -1.f : 0.f;
        wb.tok[gi] = 0;
      }
      return;
    }
    const float rn = (float)(1.0 / sqrt(yy));
    double eg = 0, gg = 0;
    for (int d = threadIdx.x; d < Df; d += blockDim.x) {
      const float e = emb[d] * rn;
      emb[d] = e;
      if (F.gemb) {
        const double g = (double)F.gemb[d];
        eg += (double)e * g;
        gg += g * g;
      }
    }
    eg = block_sum_d(eg, red);
    gg = block_sum_d(gg, red);
    if (threadIdx.x == 0) {
      const double s_size = fmin((double)P.lambda * (double)area / ((double)H * (double)W), 1.0);
      const uint32_t ac = wb.ang_cnt[gi];
      const double s_angle = ac ? (double)wb.ang_sum[gi] / (double)ac : 0.0;
      double s_sem = 1.0;
      if (F.gemb) s_sem = gg > 0 ? fmin(fmax(eg / sqrt(gg), 0.0), 1.0) : 0.0;
      const double s_dist = 0.5 + 0.5 * dbar;
      qf[0] = (float)s_size; qf[1] = (float)s_angle; qf[2] = (float)s_sem; qf[3] = (float)s_dist;
      qf[4] = (float)(((s_size * s_angle) * s_sem) * s_dist);
      qf[5] = (float)dbar;
    }
  } else if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) qf[k] = k == 4 ? -1.f : 0.f;   // geometry-only: no embedding
  }

  // ---- A5b tracking feature (R15): u = sum_p cnt_sp g_p in fp64, ascending p ----
  if (Dt > 0) {
    for (int d = threadIdx.x; d < Dt; d += blockDim.x) {
      double acc = 0.0;
      for (int i = pr0; i <= pr1; ++i)
        for (int j = pc0; j <= pc1; ++j) {
          const uint32_t c = cnt[i * Wp + j];
          if (!c) continue;
          const uint16_t b = F.track[((size_t)i * Wp + j) * Dt + d];
          const float g = __uint_as_float((uint32_t)b << 16);
          acc = __dadd_rn(acc, __dmul_rn((double)c, (double)g));
        }
      u_s[d] = acc;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const double nn = dot_pin_warp(u_s, u_s, Dt);
      double* t = wb.trk + gi * Dt;
      const bool ok = nn > 0.0;
      const double n = ok ? sqrt(nn) : 1.0;
      for (int d = threadIdx.x; d < Dt; d += 32) t[d] = ok ? __ddiv_rn(u_s[d], n) : 0.0;
      if (threadIdx.x == 0) wb.tok[gi] = ok ? 1 : 0;
    }
  }
  if (threadIdx.x == 0) wb.status[gi] = 0;
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
size_t k1_smem_bytes(int S, int W, int Wp, int rows_cap) {
  return (size_t)S * Wp * 4 + (size_t)S * 16 + (size_t)S * 4 + (size_t)K1_PLIST * 4 + (size_t)W * 4 +
         (size_t)((W + 1) & ~1) * 2 + (size_t)rows_cap * 4 + 16 + (size_t)16 * K1_THREADS * 8 + 16;
}

void launch_stage1(const WinDesc& wd, const WinBufs& wb, const Params& P, int* err, bool sem, int maxS,
                   int maxHp, int maxW, int maxWp, int maxP, int rows_cap, cudaStream_t st,
                   cudaEvent_t ev0, cudaEvent_t ev1) {
  const int n = wd.n;
  k_win_init<<<dim3(1, n), 256, 0, st>>>(wd, wb);
  debug_check(st, "k_win_init", -1);
  const size_t sm1 = k1_smem_bytes(maxS, maxW, maxWp, rows_cap);
  if (ev0) cudaEventRecord(ev0, st);
  if (sem) {
    cudaFuncSetAttribute(k_mask_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    k_mask_pass<true><<<dim3(maxHp, n), K1_THREADS, sm1, st>>>(wd, wb, P, err, rows_cap);
  } else {
    cudaFuncSetAttribute(k_mask_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    k_mask_pass<false><<<dim3(maxHp, n), K1_THREADS, sm1, st>>>(wd, wb, P, err, rows_cap);
  }
  debug_check(st, "k_mask_pass", -1);
  if (ev1) cudaEventRecord(ev1, st);
  const size_t sm2 = (size_t)maxS * (6 * 4 + 4 + 4);
  const int g2 = 64;
  if (sem) k_pairs<true><<<dim3(g2, n), K2_THREADS, sm2, st>>>(wd, wb, P, err);
  else k_pairs<false><<<dim3(g2, n), K2_THREADS, sm2, st>>>(wd, wb, P, err);
  debug_check(st, "k_pairs", -1);
  if (sem) {
    const int nch = (maxP + K3_ROWS - 1) / K3_ROWS;
    k_fbar_part<<<dim3(nch, n), 256, 0, st>>>(wd, wb, P.Df);
    k_fbar<<<dim3((P.Df + 255) / 256, n), 256, 0, st>>>(wd, wb, P.Df);
    k_resid<<<dim3((maxP + 7) / 8, n), 256, 0, st>>>(wd, wb, P.Df);
    debug_check(st, "k_fbar/k_resid", -1);
  }
  const size_t sm4 = 40 * 8 + (size_t)P.Dt * 8 + 64;
  if (sem) k_detect<true><<<dim3(maxS, n), K4_THREADS, sm4, st>>>(wd, wb, P);
  else k_detect<false><<<dim3(maxS, n), K4_THREADS, sm4, st>>>(wd, wb, P);
  debug_check(st, "k_detect", -1);
}

}  // namespace disc
