// k_frame.cu -- stage 1 of the DISC hot path: per-frame-independent work, batched over a
// window of frames.
//
//  K0  k_win_init      reset the window's per-mask accumulators
//  K1  k_mask_pass     depth -> pinned fp32 world point -> voxel key (R5) -> frame key table;
//                      every mask byte read once (16-B streaming loads): area, bbox, per-patch
//                      pixel counts, unique (s, key) pairs (|V_s|), pixel normal sums (R21)
//  K2  k_pairs         pair records for stage 2, detection AABBs, S_angle terms (Eq.3)
//  K3  k_fbar_part / k_fbar / k_resid   distinctiveness map inputs (Eq.1)
//  K4  k_filter / k_pool / k_finalize   mask filter (A1), D-weighted pooling,
//                      Q (Eq.2-3) and the tracking feature t_s (R15)
#include "disc_common.cuh"
#include "disc_launch.h"
#include "k_stage1.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace disc {

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ uint4 ld_stream16(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Streaming reads (each byte used once per window): L2 evict-first through a cache policy, so
// the window's token streams do not push the map's working set out of L2 while the
// stage-2 kernel runs beside stage 1.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ld_f4_ef(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// Table fills with streaming (evict-first) stores: the window's frame tables are cleared without
// displacing the map's working set in L2.
__global__ void k_fill_cs(uint4* p, size_t n16, uint32_t v) {
  const uint4 w = make_uint4(v, v, v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, w);
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
    wb.vs[i] = 0;
    wb.ang64[i] = 0ull;
    wb.pw[i] = 0u;
    wb.ang_cnt[i] = 0;
    wb.psum64[3 * i] = 0; wb.psum64[3 * i + 1] = 0; wb.psum64[3 * i + 2] = 0;
    wb.bbox[4 * i + 0] = INT32_MAX;
    wb.bbox[4 * i + 1] = INT32_MAX;
    wb.bbox[4 * i + 2] = -1;
    wb.bbox[4 * i + 3] = -1;
    for (int k = 0; k < 3; ++k) {
      wb.daabb[6 * i + k] = INT32_MAX;
      wb.daabb[6 * i + 3 + k] = INT32_MIN;
    }
  }
  // pooling / tracking accumulators of this frame's masks (k_pool reduces into them)
  for (size_t i = threadIdx.x + blockIdx.x * blockDim.x; i < (size_t)S * wd.Df; i += blockDim.x * gridDim.x)
    wb.emb64[(size_t)f * wb.SMAX * wd.Df + i] = 0;
  for (size_t i = threadIdx.x + blockIdx.x * blockDim.x; i < (size_t)S * wd.Dt; i += blockDim.x * gridDim.x)
    wb.trk[(size_t)f * wb.SMAX * wd.Dt + i] = 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wb.npairs[f] = 0;
    wb.rcount[f] = 0;
    wb.oor[f] = 0;
    if (f == 0) { wb.k1ctr[0] = 0; wb.k1ctr[1] = 0; *wb.s2bar = 0; }   // K1a/K1b work counters, stage-2 barrier
    wb.xmax[f] = 0.f;
  }
  // per-patch pixel counts are accumulated with atomics by K1: zero the rows this frame uses
  const int P = wd.f[f].Hp * wd.f[f].Wp;
  uint32_t* cnt = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP;
  for (int s = 0; s < S; ++s)
    for (int p = threadIdx.x + blockIdx.x * blockDim.x; p < P; p += blockDim.x * gridDim.x)
      cnt[(size_t)s * wb.PMAXP + p] = 0;
}

// ------------------------------------------------------------------------------------------
// K1: the mask pass, in three kernels (K1a/K1b persistent grids
// pulling (frame, tile) items from counters; CTAs that land on one of the first `reserve` SMs
// exit at once, leaving those SMs to stage 2):
//  K1a k_masks  streams every mask plane once (a lane owns 32 consecutive pixels of a row; the
//               four lanes 4r..4r+3 of a warp cover one tile row, so every warp load is whole
//               128-byte lines; four planes in flight): each pixel's first mask m0 and an "in a
//               second mask" bit go to HBM maps; per-patch pixel counts (R17) and bboxes.
//  K1b k_walk   lane = column, one row per step: depth -> pinned world point and key (R5), each
//               world point computed once (row below computed ahead, row above kept, left/right
//               from the adjacent lanes); a lane sums its pixel normals (R21) in registers while
//               its (m0, key) repeats down the column, and a finished run goes to the warp's
//               shared-memory queue (one ballot), drained 32 at a time into the CTA key / pair
//               tables.  Pixels in more than one mask (R9) emit their other masks per pixel.  The
//               tile's distinct pairs go to the frame's record list.
//  K1c k_dedup  one record per thread into the frame's key / pair tables (|V_s|, pair list).
// ------------------------------------------------------------------------------------------
#ifndef K1A_PERSIST
#define K1A_PERSIST 6
#endif
#ifndef K1B_PERSIST
#define K1B_PERSIST 7   // K1b CTAs per SM (A/B r02: 7 beat 8 and 6 on R and H, M1 and M2)
#endif
#ifndef K1_NFB
#define K1_NFB 4   // bit-packed mask words in flight per lane (K1a; measured H: 4 139, 8 150, 16 219 us per window)
#endif
#ifndef K1_NF
#define K1_NF 4   // mask planes in flight per lane (K1a)
#endif
constexpr int K1_THREADS = 128;
constexpr int K1_WARPS = K1_THREADS / 32;
constexpr int K1_TW = 32;                                 // tile columns per warp
// output columns per warp: 30 with normals (lanes 0 and 31 compute the neighbour columns), else 32
__host__ __device__ constexpr int k1_cols_out(bool sem) { return sem ? K1_TW - 2 : K1_TW; }
constexpr int K1_TILE_H = 32;
constexpr int K1_KT = K1_PT / 2;                          // CTA key table slots (2 pair slots each)
constexpr int K1_PLIST = 512;
constexpr int K1_KT_PROBES = 16;                           // CTA key-table probe bound
constexpr uint32_t K1_Q = 64;
constexpr uint32_t K1C_PL = 1024;                        // k_dedup per-block pair list
#ifndef K1C_BLOCKS
#define K1C_BLOCKS 64   // K1c blocks per frame
#endif                             // k_walk per-warp run queue
constexpr uint16_t K1_NOKEY = 0xFFFF;

#ifndef K1_MASK_L2
#define K1_MASK_L2 0   // 0: L2 evict_first, 1: default policy, 2: default + 256-B prefetch
#endif
__device__ __forceinline__ void ld_stream32(const uint8_t* p, uint32_t r[8]) {
#if K1_MASK_L2 == 0
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
#elif K1_MASK_L2 == 1
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
#endif
}
// (bit-packed mask words) read-only path, no L1 allocation, L2 evict-first through a cache policy
// (the .L2::evict_first qualifier form needs a 32-byte vector)
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
// 4 mask bits -> 4 bytes of 0 / 1 (bit i -> byte i; the shifted copies of the nibble never overlap)
__device__ __forceinline__ uint32_t nib_bytes(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }
__device__ __forceinline__ uint4 ld_mask16(const uint8_t* p) {
  uint4 r;
#if K1_MASK_L2 == 1
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#endif
  return r;
}

__device__ __forceinline__ uint32_t range_bits(int a, int b) {   // bits [a, b), 0 <= a < b <= 32
  return (b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u)) & ~((1u << a) - 1u);
}

// Stage 2's persistent grid (cooperative, one CTA per SM) lands where the hardware puts it.  While
// one runs, a stage-1 CTA keeps off exactly the SMs it occupies (s2sm: its CTAs' SM bits and count);
// otherwise off SMs [0, reserve), which stays free for the next stage-2 launch.  (A fixed [0, reserve)
// alone left stage 1 the SMs >= reserve minus the stage-2 CTAs placed there: ~16 instead of 48 SMs
// when a stage-2 grid started first and spread over the GPU.)
__device__ __forceinline__ bool on_reserved_sm(int reserve, const uint32_t* s2sm) {
  if (reserve <= 0) return false;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (*(volatile const uint32_t*)(s2sm + 5) > 0) return (*(volatile const uint32_t*)(s2sm + (sm >> 5)) >> (sm & 31)) & 1u;
  return (int)sm < reserve;
}

// next (frame, tile) item of a persistent K1 grid; CTA-uniform, -1 when done
__device__ __forceinline__ int next_item(uint32_t* ctr, uint32_t total, uint32_t* item_s) {
  __syncthreads();   // the previous item's shared state is no longer read
  if (threadIdx.x == 0) *item_s = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t it = *item_s;
  return it < total ? (int)it : -1;
}

// ---- K1a ----------------------------------------------------------------------------------
// The frame is taken as one flat pixel array: lane l of an item owns the 32-byte sector
// [32 k, 32 k + 32) of every mask plane (k = item * 128 + thread), so a warp load is 1 KB of
// consecutive, aligned bytes.  A sector may cross row ends; rows and patches are recovered per
// sector only for the planes that touch it.
constexpr int K1A_SECT = K1_THREADS;   // sectors per item

// BM: mask planes of the window's frames -- 0 all byte planes, 1 all bit-packed, 2 mixed (per frame)
template <bool VEC, int BM>
__global__ void __launch_bounds__(K1_THREADS, K1A_PERSIST) k_masks(WinDesc wd, WinBufs wb, int items_f, int reserve,
                                                                  int ablate) {
  if (on_reserved_sm(reserve, wb.s2sm)) return;
  extern __shared__ int32_t bb_s[];          // [S][4] umin, vmin, umax, vmax
  __shared__ uint32_t item_s;
  const uint32_t total = (uint32_t)items_f * (uint32_t)wd.n;
  for (int it; (it = next_item(wb.k1ctr, total, &item_s)) >= 0;) {
    const int f = it / items_f, item = it % items_f;   // frame-major
    const FrameDesc& F = wd.f[f];
    const int H = F.H, W = F.W, S = F.S, Hp = F.Hp, Wp = F.Wp;
    const int64_t HW = (int64_t)H * W;
    if ((int64_t)item * K1A_SECT * 32 >= HW) continue;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      bb_s[4 * i + 0] = INT32_MAX; bb_s[4 * i + 1] = INT32_MAX;
      bb_s[4 * i + 2] = -1; bb_s[4 * i + 3] = -1;
    }
    __syncthreads();
    const int64_t p0 = ((int64_t)item * K1A_SECT + threadIdx.x) * 32;   // first pixel of the sector
    const int nv = p0 < HW ? (int)min((int64_t)32, HW - p0) : 0;
    const uint32_t inb = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    // 32-bit index arithmetic: H, W <= 16384 (validated), so every product below is < 2^31
    const int v0 = nv ? (int)((uint32_t)p0 / (uint32_t)W) : 0;
    const int u0 = nv ? (int)p0 - v0 * W : 0;
    uint32_t* cnt_f = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP;
    // bit-packed planes: the sector is exactly word p0/32 of the plane (one 4-byte load instead of 32),
    // kept raw in w[0] until used
    const bool bits = BM == 1 || (BM == 2 && F.mbits != nullptr);
    const uint32_t* mbp = bits ? F.mbits + (p0 >> 5) : nullptr;
    const size_t wpl = ((size_t)HW + 31) >> 5;
    auto load = [&](int s, uint32_t w[8]) {
      const uint8_t* mp = F.masks + (size_t)s * HW + p0;
      if (VEC) {
        ld_stream32(mp, w);
      } else {
        for (int t = 0; t < 8; ++t) {
          uint32_t x = 0;
          for (int bq = 0; bq < 4; ++bq)
            if (inb & (1u << (4 * t + bq))) x |= (uint32_t)(mp[4 * t + bq] != 0) << (8 * bq);
          w[t] = x;
        }
      }
    };
    // the sector's row / patch segmentation, once for all planes: segment starts (bit j), their
    // patch indices (up to K1A_NSEG), and the row break jb (W >= 32: at most two rows)
    constexpr int K1A_NSEG = 8;
    uint32_t segbits = 0;
    int pidx[K1A_NSEG];
    int nseg = 0;
    bool fast = W >= 32;
    {
      int j = 0, v = v0, u = u0;
      while (j < nv) {
        const int len = min(W - u, nv - j);
        const int prow = (v * Hp) / H * Wp;
        int pcol = (u * Wp) / W;
        int jj = j, uu = u;
        while (jj < j + len) {
          const int ub = ((pcol + 1) * W + Wp - 1) / Wp;   // first u of the next patch column
          const int l2 = min(j + len - jj, ub - uu);
          segbits |= 1u << jj;
#pragma unroll
          for (int k = 0; k < K1A_NSEG; ++k)
            if (k == nseg) pidx[k] = prow + pcol;
          ++nseg;
          jj += l2; uu += l2; ++pcol;
        }
        j += len; ++v; u = 0;
      }
      if (nseg > K1A_NSEG) fast = false;
    }
    const int jb = u0 + nv > W ? W - u0 : 32;   // first pixel of the second row
    const uint32_t rowA = jb >= 32 ? 0xFFFFFFFFu : ((1u << jb) - 1u);
    uint32_t m0[8], ovf = 0, unset_b = 0xFFFFFFFFu;   // (unset_b: bit-packed path, pixels without a mask yet)
#pragma unroll
    for (int t = 0; t < 8; ++t) m0[t] = 0xFFFFFFFFu;   // no mask yet
    const int Sl = (nv && !(ablate & 1)) ? S : 0;
    // per-patch pixel counts (O5, regardless of depth, R17) and bbox of mask s over the sector's
    // pixels `set` (bit j = pixel p0 + j)
    auto tally = [&](int s, uint32_t set) {
      if (fast) {   // per-patch pixel counts (O5, regardless of depth, R17) and bbox
        uint32_t sb = segbits;
#pragma unroll
        for (int k = 0; k < K1A_NSEG; ++k) {
          if (k >= nseg) break;
          const int a0 = __ffs(sb) - 1;
          sb &= sb - 1;
          const int b0 = sb ? __ffs(sb) - 1 : 32;
          const int cn = __popc(set & range_bits(a0, b0));
          if (cn) atomicAdd(&cnt_f[(size_t)s * wb.PMAXP + pidx[k]], (uint32_t)cn);
        }
        const uint32_t sa = set & rowA, sb2 = set & ~rowA;
        if (sa) {
          atomicMin(&bb_s[4 * s + 0], u0 + __ffs(sa) - 1);
          atomicMax(&bb_s[4 * s + 2], u0 + 31 - __clz(sa));
          atomicMin(&bb_s[4 * s + 1], v0);
          atomicMax(&bb_s[4 * s + 3], v0);
        }
        if (sb2) {
          atomicMin(&bb_s[4 * s + 0], __ffs(sb2) - 1 - jb);
          atomicMax(&bb_s[4 * s + 2], 31 - __clz(sb2) - jb);
          atomicMin(&bb_s[4 * s + 1], v0 + 1);
          atomicMax(&bb_s[4 * s + 3], v0 + 1);
        }
        return;
      }
      // general: row segments of the sector, and patch segments inside them
      int j = 0, v = v0, u = u0;
      while (j < nv) {
        const int len = min(W - u, nv - j);
        const uint32_t rowb = set & range_bits(j, j + len);
        if (rowb) {
          const int prow = (v * Hp) / H * Wp;
          int pcol = (u * Wp) / W;
          int jj = j, uu = u;
          while (jj < j + len) {
            const int ub = ((pcol + 1) * W + Wp - 1) / Wp;   // first u of the next patch column
            const int l2 = min(j + len - jj, ub - uu);
            const int cn = __popc(set & range_bits(jj, jj + l2));
            if (cn) atomicAdd(&cnt_f[(size_t)s * wb.PMAXP + prow + pcol], (uint32_t)cn);
            jj += l2; uu += l2; ++pcol;
          }
          atomicMin(&bb_s[4 * s + 0], u + (__ffs(rowb) - 1 - j));
          atomicMax(&bb_s[4 * s + 2], u + (31 - __clz(rowb) - j));
          atomicMin(&bb_s[4 * s + 1], v);
          atomicMax(&bb_s[4 * s + 3], v);
        }
        j += len; ++v; u = 0;
      }
    };
    if (BM != 0 && bits) {
      // bit-packed planes: one word per plane and sector, K1_NFB planes in flight per lane (4-byte
      // loads: a deeper ring than the byte planes' 32-byte ones for the same bytes in flight); the
      // first-mask bytes are touched only for pixels meeting their first mask
      uint32_t rb[K1_NFB];
      const uint64_t pol = policy_evict_first();
#pragma unroll
      for (int k = 0; k < K1_NFB; ++k) rb[k] = k < Sl ? ld_stream_u32(mbp + (size_t)k * wpl, pol) : 0u;
      for (int s0 = 0; s0 < Sl; s0 += K1_NFB) {
#pragma unroll
        for (int k = 0; k < K1_NFB; ++k) {
          const int s = s0 + k;
          if (s >= Sl) break;
          const uint32_t set = rb[k] & inb;   // (the raw word: consuming a load at its refill would wait for it)
          if (s + K1_NFB < Sl) rb[k] = ld_stream_u32(mbp + (size_t)(s + K1_NFB) * wpl, pol);   // refill
          if (!set) continue;
          const uint32_t fresh = set & unset_b;
          ovf |= set & ~unset_b;
          unset_b &= ~set;
          if (fresh) {
            const uint32_t splat = (uint32_t)s * 0x01010101u;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const uint32_t fm = nib_bytes((fresh >> (4 * t)) & 0xFu) * 0xFFu;
              m0[t] = (m0[t] & ~fm) | (splat & fm);
            }
          }
          tally(s, set);
        }
      }
    } else if (BM != 1) {
      uint32_t buf[K1_NF][8];
#pragma unroll
      for (int k = 0; k < K1_NF; ++k)
        if (k < Sl) load(k, buf[k]);
      for (int s0 = 0; s0 < Sl; s0 += K1_NF) {
#pragma unroll
        for (int k = 0; k < K1_NF; ++k) {
          const int s = s0 + k;
          if (s >= Sl) break;
          uint32_t* w = buf[k];
          if ((w[0] | w[1] | w[2] | w[3] | w[4] | w[5] | w[6] | w[7]) == 0) {
            if (s + K1_NF < Sl) load(s + K1_NF, buf[k]);   // refill the ring slot
            continue;
          }
          uint32_t set = 0;
          const uint32_t splat = (uint32_t)s * 0x01010101u;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint32_t sb = __vcmpne4(w[t], 0u);                // 0xFF where the pixel is in s
            set |= (((sb & 0x08040201u) * 0x01010101u) >> 24) << (4 * t);
            const uint32_t unset = __vcmpeq4(m0[t], 0xFFFFFFFFu);   // 0xFF where no mask yet
            const uint32_t fresh = sb & unset, again = sb & ~unset;
            m0[t] = (m0[t] & ~fresh) | (splat & fresh);
            ovf |= (((again & 0x08040201u) * 0x01010101u) >> 24) << (4 * t);
          }
          if (s + K1_NF < Sl) load(s + K1_NF, buf[k]);   // refill the ring slot
          set &= inb;
          if (set) tally(s, set);
        }
      }
    }
    if (nv) {   // first-mask map, u16 per pixel: m0 | (in a second mask) << 8 (flat, 64-B aligned)
      uint16_t* mo = wb.m0map + (size_t)f * wb.MPIX + p0;
      if (VEC) {
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
          uint32_t q[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t w = m0[t + h], ob = ovf >> (4 * (t + h));
            q[2 * h] = __byte_perm(w, 0, 0x4140) | ((ob & 1u) << 8) | (((ob >> 1) & 1u) << 24);
            q[2 * h + 1] = __byte_perm(w, 0, 0x4342) | (((ob >> 2) & 1u) << 8) | (((ob >> 3) & 1u) << 24);
          }
          __stcs((uint4*)mo + t / 2, make_uint4(q[0], q[1], q[2], q[3]));   // streaming: read once by K1b
        }
      } else {
        for (int j = 0; j < nv; ++j)
          mo[j] = (uint16_t)(((m0[j >> 2] >> (8 * (j & 3))) & 0xFFu) | (((ovf >> j) & 1u) << 8));
      }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
      if (bb_s[4 * s + 2] < 0) continue;   // mask absent from this item
      const size_t gi = (size_t)f * wb.SMAX + s;
      atomicMin(&wb.bbox[4 * gi + 0], bb_s[4 * s + 0]);
      atomicMin(&wb.bbox[4 * gi + 1], bb_s[4 * s + 1]);
      atomicMax(&wb.bbox[4 * gi + 2], bb_s[4 * s + 2]);
      atomicMax(&wb.bbox[4 * gi + 3], bb_s[4 * s + 3]);
    }
  }
}

// ---- K1b ----------------------------------------------------------------------------------
template <bool SEM>
__global__ void __launch_bounds__(K1_THREADS, K1B_PERSIST) k_walk(WinDesc wd, WinBufs wb, Params P, int* err,
                                                                 int tiles_x, int reserve, int ablate) {
  if (on_reserved_sm(reserve, wb.s2sm)) return;
  extern __shared__ uint32_t vs_s[];                        // [S] |V_s| contributions
  __shared__ unsigned long long kt[K1_KT];                  // CTA key table
  __shared__ uint32_t ptc[2 * K1_KT];                       // pair slots 2 li, 2 li + 1: s or EMPTY
  __shared__ uint32_t pl_s[K1_PLIST];
  __shared__ float yb_s[K1_TILE_H + 2];                     // row r <-> v = vt0 - 1 + r (R5)
  __shared__ float4 pose_s[3];                              // pose rows (R5): re-read, not held in registers
  __shared__ unsigned long long qk[K1_WARPS][K1_Q];          // per-warp queue of finished runs: key,
  __shared__ uint32_t qs[K1_WARPS][K1_Q];                    //   mask index,
  __shared__ float qv[K1_WARPS][SEM ? K1_Q : 1][3];          //   normal sum
  __shared__ uint32_t item_s, slot_s, npl_s, oor_s, base_s, rc_s, rb_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (SEM && threadIdx.x == 0) {   // a scratch block of this SM for the tiles' normal sums
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    uint32_t* w = wb.k1slot + sm;
    for (;;) {
      const uint32_t freeb = ~*(volatile uint32_t*)w & ((1u << K1_SLOTS_PER_SM) - 1u);
      if (!freeb) continue;
      const uint32_t b = __ffs(freeb) - 1;
      if (!(atomicOr(w, 1u << b) & (1u << b))) { slot_s = sm * K1_SLOTS_PER_SM + b; break; }
    }
    __threadfence();
  }
  const float rv = P.r;
  const float rinv = 1.0f / P.r;   // only used by floor_div_pinned's exact fast path
  const uint32_t total = (uint32_t)tiles_x * (uint32_t)wd.n;
  for (int it; (it = next_item(wb.k1ctr + 1, total, &item_s)) >= 0;) {
    const int f = it / tiles_x, tile = it % tiles_x;
    const FrameDesc& F = wd.f[f];
    const int H = F.H, W = F.W, S = F.S;
    constexpr int TWO = k1_cols_out(SEM), TILE_W = K1_WARPS * TWO;
    const int ntx = (W + TILE_W - 1) / TILE_W, nty = (H + K1_TILE_H - 1) / K1_TILE_H;
    if (tile >= ntx * nty) continue;
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int ut0 = tx * TILE_W, vt0 = ty * K1_TILE_H;
    NSum* nscr = SEM ? wb.k1scr + (size_t)slot_s * K1_PT : nullptr;
    for (int i = threadIdx.x; i < S; i += blockDim.x) vs_s[i] = 0;
    for (int i = threadIdx.x; i < K1_KT; i += blockDim.x) kt[i] = KEY_EMPTY;
    for (int i = threadIdx.x; i < 2 * K1_KT; i += blockDim.x) ptc[i] = U32_EMPTY;
    for (int r = threadIdx.x; r < K1_TILE_H + 2; r += blockDim.x)
      yb_s[r] = __fdiv_rn(__fsub_rn((float)(vt0 - 1 + r), F.cy), F.fy);
    if (threadIdx.x < 3)
      pose_s[threadIdx.x] = make_float4(F.pose[4 * threadIdx.x], F.pose[4 * threadIdx.x + 1], F.pose[4 * threadIdx.x + 2],
                                        F.pose[4 * threadIdx.x + 3]);
    if (threadIdx.x == 0) { npl_s = 0; oor_s = 0; rc_s = 0; }
    __syncthreads();

    const uint32_t tmask = (uint32_t)wb.PC - 1;
    unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
    uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
    NSum* nsum = wb.nsum + (size_t)f * wb.PC;
    // CTA key table -> local key index; at most K1_KT_PROBES probes, so a table that far views
    // (up to a voxel per pixel) fill up fails fast and the item takes the record list
    auto kt_insert = [&](uint64_t key) -> uint16_t {
      uint32_t h = (uint32_t)mix64(key) & (K1_KT - 1);
      for (int probe = 0; probe < K1_KT_PROBES; ++probe) {
        const unsigned long long cur = kt[h];
        if (cur == key) return (uint16_t)h;
        if (cur == KEY_EMPTY) {
          const unsigned long long old = atomicCAS(&kt[h], KEY_EMPTY, (unsigned long long)key);
          if (old == KEY_EMPTY || old == key) return (uint16_t)h;
        }
        h = (h + 1) & (K1_KT - 1);
      }
      return K1_NOKEY;
    };
    auto global_insert = [&](uint64_t key, uint32_t s) -> uint32_t {
      const uint32_t kslot = ktab_insert(ktab, tmask, key, err);
      if (kslot == U32_EMPTY) return U32_EMPTY;
      bool fresh = false;
      const uint32_t pslot = ptab_insert(ptab, tmask, (s << 24) | kslot, &fresh, err);
      if (pslot != U32_EMPTY && fresh) {
        atomicAdd(&vs_s[s], 1u);
        const uint32_t li = atomicAdd(&npl_s, 1u);
        if (li < K1_PLIST) {
          pl_s[li] = pslot;
        } else {
          const uint32_t gi2 = atomicAdd(&wb.npairs[f], 1u);
          if (gi2 < (uint32_t)wb.PMAX) wb.plist[(size_t)f * wb.PMAX + gi2] = pslot;
          else raise_err(err, DERR_FRAME_PAIRS);
        }
      }
      return pslot;
    };
    // one (s, key) item: CTA key table -> local index li; the pair is slot 2 li or 2 li + 1 (a
    // voxel rarely meets more than two masks in one tile); otherwise straight to the frame tables
    // one (s, key) item into the CTA tables; false when they are full (the caller spills it)
    auto emit_cta = [&](uint32_t s, uint64_t key, float n0, float n1, float n2) -> bool {
      const uint16_t li = kt_insert(key);
      int ps = -1;
      if (li != K1_NOKEY) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          uint32_t* c = &ptc[2 * li + jj];
          uint32_t cur = *c;
          if (cur == U32_EMPTY) {
            cur = atomicCAS(c, U32_EMPTY, s);
            if (cur == U32_EMPTY) cur = s;
          }
          if (cur == s) { ps = 2 * li + jj; break; }
        }
      }
      if (ps < 0) return false;
      if (SEM && (n0 != 0.f || n1 != 0.f || n2 != 0.f)) nsum_add(&nscr[ps], n0, n1, n2);
      return true;
    };
    auto emit = [&](uint32_t s, uint64_t key, float n0, float n1, float n2) -> int {
      const uint16_t li = kt_insert(key);
      int ps = -1;
      if (li != K1_NOKEY) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          uint32_t* c = &ptc[2 * li + jj];
          uint32_t cur = *c;
          if (cur == U32_EMPTY) {
            cur = atomicCAS(c, U32_EMPTY, s);
            if (cur == U32_EMPTY) cur = s;
          }
          if (cur == s) { ps = 2 * li + jj; break; }
        }
      }
      const bool hasn = SEM && (n0 != 0.f || n1 != 0.f || n2 != 0.f);
      if (ps >= 0) {
        if (hasn) nsum_add(&nscr[ps], n0, n1, n2);
        return ps;
      }
      const uint32_t g = global_insert(key, s);
      if (hasn && g != U32_EMPTY) nsum_add(&nsum[g], n0, n1, n2);
      return -1;
    };

    // ---- walk: lane = column, one row per step; with normals (SEM) a warp's 32 lanes cover 30
    // output columns, lanes 0 and 31 being the left / right neighbour columns (no items) ----
    const int u = ut0 + warp * TWO + lane - (SEM ? 1 : 0);
    const bool out_lane = !SEM || (lane >= 1 && lane <= 30);
    const int rows = min(K1_TILE_H, H - vt0);
    uint32_t my_oor = 0;
    if (!(ablate & 2) && ut0 + warp * TWO < W) {
      const bool col_on = u >= 0 && u < W;
      const float xa = col_on ? __fdiv_rn(__fsub_rn((float)u, F.cx), F.fx) : 0.f;   // R5
      const float* dcol = F.depth + (col_on ? u : 0);
      const uint16_t* mcol = wb.m0map + (size_t)f * wb.MPIX + (col_on ? u : 0);
      const bool m_on = col_on && out_lane;   // first-mask entries of the output columns only
      auto wpt = [&](float d, float x, float yb, float p[3]) -> bool {
        if (!depth_valid(d, P)) return false;
        const float xc = __fmul_rn(x, d), yc = __fmul_rn(yb, d), zc = d;
        const float4 a = pose_s[0], b = pose_s[1], c = pose_s[2];
        p[0] = __fmaf_rn(a.x, xc, __fmaf_rn(a.y, yc, __fmaf_rn(a.z, zc, a.w)));
        p[1] = __fmaf_rn(b.x, xc, __fmaf_rn(b.y, yc, __fmaf_rn(b.z, zc, b.w)));
        p[2] = __fmaf_rn(c.x, xc, __fmaf_rn(c.y, yc, __fmaf_rn(c.z, zc, c.w)));
        return true;
      };
      auto drow = [&](const float* base, bool on, int vv) -> float {   // 0 (invalid) off-image
        const float d = __ldg(base + min(max(vv, 0), H - 1) * W);   // in-bounds address, no branch
        return (on && (unsigned)vv < (unsigned)H) ? d : 0.f;
      };
      // R6 range test alone, for pixels in no mask (only key_out_of_range needs them): exact
      // fast accept when |x| <= 2^19 r, else the pinned key
      auto in_range = [&](const float p[3]) -> bool {
        const float lim = 524288.0f * rv;
        if (fabsf(p[0]) <= lim && fabsf(p[1]) <= lim && fabsf(p[2]) <= lim) return true;
        uint64_t k;
        return point_key_fast(p, rv, rinv, k);
      };
      float pu[3] = {0.f, 0.f, 0.f}, pc[3] = {0.f, 0.f, 0.f};
      bool vu = SEM ? wpt(drow(dcol, col_on, vt0 - 1), xa, yb_s[0], pu) : false;
      bool vc = wpt(drow(dcol, col_on, vt0), xa, yb_s[1], pc);
      uint32_t mv_c = m_on ? mcol[vt0 * W] : 0xFFu;   // m0 | overlap << 8
      uint64_t kc = KEY_EMPTY;
      bool kvc = vc && ((mv_c & 0xFFu) != 0xFFu ? point_key_fast(pc, rv, rinv, kc) : in_range(pc));
      float d_dn = drow(dcol, col_on, vt0 + 1);
      // the lane's pending item (rows repeat voxels)
      uint32_t qn = 0;   // records in the warp's queue (warp-uniform)
      // the queue into the CTA tables; items they cannot hold (far views: up to a voxel per pixel)
      // go to the frame's record list for K1c (one reservation per warp), and only past its
      // capacity into the frame tables from here
      auto drain = [&]() {
        __syncwarp();
        for (uint32_t i0 = 0; i0 < qn; i0 += 32) {
          const uint32_t i = i0 + lane;
          uint32_t s = 0;
          unsigned long long key = 0;
          float a = 0.f, b = 0.f, c = 0.f;
          bool spill = false;
          if (i < qn) {
            s = qs[warp][i];
            key = qk[warp][i];
            if (SEM) { a = qv[warp][i][0]; b = qv[warp][i][1]; c = qv[warp][i][2]; }
            spill = !emit_cta(s, key, a, b, c);
          }
          const unsigned sm = __ballot_sync(0xffffffffu, spill);
          if (sm) {
            const int ld = __ffs(sm) - 1;
            uint32_t rb = 0;
            if (lane == ld) rb = atomicAdd(&wb.rcount[f], (uint32_t)__popc(sm));
            rb = __shfl_sync(0xffffffffu, rb, ld);
            if (spill) {
              const uint32_t r = rb + __popc(sm & ((1u << lane) - 1u));
              if (r < (uint32_t)wb.RCAP) {
                const size_t o = (size_t)f * wb.PMAX + r;
                __stcg(&wb.rkey[o], key);
                __stcg(&wb.rs[o], s);
                if (SEM) wb.rn[o] = NSum{llrint((double)a * NSCALE), llrint((double)b * NSCALE), llrint((double)c * NSCALE), 0};
              } else {
                const uint32_t g = global_insert(key, s);
                if (SEM && g != U32_EMPTY && (a != 0.f || b != 0.f || c != 0.f)) nsum_add(&nsum[g], a, b, c);
              }
            }
          }
        }
        __syncwarp();
        qn = 0;
      };
      uint64_t ck = KEY_EMPTY;
      uint32_t cs = 0xFFFFFFFFu;
      float pn0 = 0.f, pn1 = 0.f, pn2 = 0.f;
      // running row pointers (no per-row index arithmetic): depth two rows ahead, first-mask
      // entry one row ahead; a pointer past the image is never dereferenced
      const float* dp = dcol + (int64_t)(vt0 + 2) * W;
      const uint16_t* mp = mcol + (int64_t)(vt0 + 1) * W;
      const int lim2 = col_on ? H - vt0 - 2 : -1;   // rr < lim2: row vv + 2 exists (and the column)
      for (int rr = 0; rr < rows; ++rr) {
        const int vv = vt0 + rr;
        // the next row's loads go out before this row's arithmetic
        const float d_dn2 = rr < lim2 ? __ldcs(dp) : 0.f;   // streaming (evict-first) reads
        const bool more = rr + 1 < rows;
        const uint32_t mv_n = (m_on && more) ? (uint32_t)__ldcs(mp) : 0xFFu;
        dp += W; mp += W;
        const float ybn = yb_s[rr + 2];
        float pd[3] = {0.f, 0.f, 0.f};
        const bool vd = wpt(d_dn, xa, ybn, pd);
        const uint32_t m = mv_c & 0xFFu;
        if (out_lane && vc && !kvc) my_oor++;
        const bool item = m != 0xFFu && kvc;   // (m is 0xFF in the neighbour lanes)
        float n0 = 0.f, n1 = 0.f, n2 = 0.f;
        if (SEM) {
          float pl[3], pr[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            pl[a] = __shfl_up_sync(0xffffffffu, pc[a], 1);
            pr[a] = __shfl_down_sync(0xffffffffu, pc[a], 1);
          }
          const unsigned vb = __ballot_sync(0xffffffffu, vc);
          const bool vl = (vb >> ((lane - 1) & 31)) & 1u, vr = (vb >> ((lane + 1) & 31)) & 1u;
          // R21 with 4 valid neighbours (off-image neighbours read depth 0 = invalid)
          if (item && vl && vr && vu && vd) {
            const float a0 = pr[0] - pl[0], a1 = pr[1] - pl[1], a2 = pr[2] - pl[2];
            const float b0 = pd[0] - pu[0], b1 = pd[1] - pu[1], b2 = pd[2] - pu[2];
            n0 = a1 * b2 - a2 * b1;
            n1 = a2 * b0 - a0 * b2;
            n2 = a0 * b1 - a1 * b0;
            const float o = n0 * (pose_s[0].w - pc[0]) + n1 * (pose_s[1].w - pc[1]) + n2 * (pose_s[2].w - pc[2]);
            if (o < 0.f) { n0 = -n0; n1 = -n1; n2 = -n2; }
          }
        }
        // vertical runs: a lane's item accumulates in registers while it repeats the same (s, key)
        // down the rows; a finished run is appended to the warp's queue (one ballot, no divergent
        // table work per row) and the queue is drained into the CTA tables 32 records at a time
        const bool same = item && kc == ck && m == cs;
        const bool push = item && !same && cs != 0xFFFFFFFFu;
        const unsigned pm = __ballot_sync(0xffffffffu, push);
        if (pm) {
          if (push) {
            const uint32_t pos = qn + __popc(pm & ((1u << lane) - 1u));
            qk[warp][pos] = ck;
            qs[warp][pos] = cs;
            if (SEM) { qv[warp][pos][0] = pn0; qv[warp][pos][1] = pn1; qv[warp][pos][2] = pn2; }
          }
          qn += __popc(pm);
          if (qn > K1_Q - 32) { drain(); }
        }
        if (item) {
          if (same) { pn0 += n0; pn1 += n1; pn2 += n2; }
          else { ck = kc; cs = m; pn0 = n0; pn1 = n1; pn2 = n2; }
          if (mv_c >> 8) {   // other masks of this pixel (R9), per pixel
            const size_t pix = (size_t)vv * W + u;
            for (int s2 = (int)m + 1; s2 < S; ++s2)
              if (mask_at(F, s2, pix)) emit((uint32_t)s2, kc, n0, n1, n2);
          }
        }
        pu[0] = pc[0]; pu[1] = pc[1]; pu[2] = pc[2]; vu = vc;
        pc[0] = pd[0]; pc[1] = pd[1]; pc[2] = pd[2]; vc = vd;
        kc = KEY_EMPTY;
        kvc = vc && ((mv_n & 0xFFu) != 0xFFu ? point_key_fast(pc, rv, rinv, kc) : in_range(pc));
        d_dn = d_dn2; mv_c = mv_n;
      }
      {
        const bool push = cs != 0xFFFFFFFFu;
        const unsigned pm = __ballot_sync(0xffffffffu, push);
        if (push) {
          const uint32_t pos = qn + __popc(pm & ((1u << lane) - 1u));
          qk[warp][pos] = ck;
          qs[warp][pos] = cs;
          if (SEM) { qv[warp][pos][0] = pn0; qv[warp][pos][1] = pn1; qv[warp][pos][2] = pn2; }
        }
        qn += __popc(pm);
        drain();
      }
    }
    if (my_oor) atomicAdd(&oor_s, my_oor);
    if (SEM) __threadfence();   // this thread's normal reductions before the reads below
    __syncthreads();
    // ---- the tile's distinct (s, key) items -> the frame's record list (K1c inserts them into
    // the frame tables with many inserts in flight); a full list sends the tile to the tables here
    uint32_t mine = 0;
    for (int i = threadIdx.x; i < 2 * K1_KT; i += blockDim.x) mine += ptc[i] != U32_EMPTY;
    const uint32_t roff = mine ? atomicAdd(&rc_s, mine) : 0;
    __syncthreads();
    if (threadIdx.x == 0) rb_s = rc_s ? atomicAdd(&wb.rcount[f], rc_s) : 0;
    __syncthreads();
    // past RCAP: this tile inserts its items itself and blanks its reserved records below RCAP
    const bool direct = rb_s + rc_s > (uint32_t)wb.RCAP;
    uint32_t r = rb_s + roff;
    for (int i = threadIdx.x; i < 2 * K1_KT; i += blockDim.x) {
      const uint32_t s = ptc[i];
      if (s == U32_EMPTY) continue;
      NSum nn{0, 0, 0, 0};
      if (SEM) {
        nn.x = __ldcg(&nscr[i].x); nn.y = __ldcg(&nscr[i].y); nn.z = __ldcg(&nscr[i].z);
        if (nn.x || nn.y || nn.z) nscr[i] = NSum{0, 0, 0, 0};
      }
      if (!direct) {
        DBOUND(r < (uint32_t)wb.RCAP, err);
        const size_t o = (size_t)f * wb.PMAX + r++;
        __stcg(&wb.rkey[o], kt[i >> 1]);
        __stcg(&wb.rs[o], s);
        if (SEM) wb.rn[o] = nn;
      } else {
        if (r < (uint32_t)wb.RCAP) __stcg(&wb.rkey[(size_t)f * wb.PMAX + r], (unsigned long long)KEY_EMPTY);
        ++r;
        const uint32_t g = global_insert(kt[i >> 1], s);
        if (SEM && g != U32_EMPTY) nsum_add_fx(&nsum[g], nn.x, nn.y, nn.z);
      }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x)
      if (vs_s[s]) atomicAdd(&wb.vs[(size_t)f * wb.SMAX + s], vs_s[s]);
    const uint32_t n = min(npl_s, (uint32_t)K1_PLIST);
    if (threadIdx.x == 0) {
      base_s = n ? atomicAdd(&wb.npairs[f], n) : 0;
      if (oor_s) atomicAdd(&wb.oor[f], (unsigned long long)oor_s);
    }
    __syncthreads();
    if (base_s + n > (uint32_t)wb.PMAX) {
      if (threadIdx.x == 0) raise_err(err, DERR_FRAME_PAIRS);
    } else {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) wb.plist[(size_t)f * wb.PMAX + base_s + i] = pl_s[i];
    }
  }
  if (SEM && threadIdx.x == 0) {
    __threadfence();
    atomicAnd(wb.k1slot + slot_s / K1_SLOTS_PER_SM, ~(1u << (slot_s % K1_SLOTS_PER_SM)));
  }
}

// ---- K1c ----------------------------------------------------------------------------------
// The tiles' (s, key) records -> the frame's key / pair tables (A3): one record per thread, so
// thousands of the dependent L2 compare-and-swap chains are in flight at once (inside K1b they
// stalled the whole CTA at the end of every tile).  Fresh pairs count into |V_s| and the pair list.
template <bool SEM>
__global__ void __launch_bounds__(256) k_dedup(WinDesc wd, WinBufs wb, int* err) {
  extern __shared__ uint32_t vsd_s[];   // [S] fresh pairs per mask
  __shared__ uint32_t pl_s[K1C_PL];     // the block's fresh pair slots
  __shared__ uint32_t npl_s, base_s;
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const int S = wd.f[f].S;
  for (int i = threadIdx.x; i < S; i += blockDim.x) vsd_s[i] = 0;
  if (threadIdx.x == 0) npl_s = 0;
  __syncthreads();
  const uint32_t n = min(wb.rcount[f], (uint32_t)wb.RCAP);
  const uint32_t tmask = (uint32_t)wb.PC - 1;
  unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
  NSum* nsum = wb.nsum + (size_t)f * wb.PC;
  for (uint32_t b = blockIdx.x * blockDim.x; b < n; b += gridDim.x * blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    bool fresh = false;
    uint32_t pslot = U32_EMPTY;
    if (i < n) {
      const size_t o = (size_t)f * wb.PMAX + i;
      const unsigned long long key = __ldcs(&wb.rkey[o]);
      const uint32_t s = __ldcs(&wb.rs[o]);
      const uint32_t kslot = key == KEY_EMPTY ? U32_EMPTY : ktab_insert(ktab, tmask, key, err);
      if (kslot != U32_EMPTY) pslot = ptab_insert(ptab, tmask, (s << 24) | kslot, &fresh, err);
      if (SEM && pslot != U32_EMPTY) {
        const NSum nn = wb.rn[o];
        nsum_add_fx(&nsum[pslot], nn.x, nn.y, nn.z);
      }
      if (fresh) atomicAdd(&vsd_s[s], 1u);
    }
    if (fresh) {   // the block's list first (one global reservation per block), else the frame's
      const uint32_t li = atomicAdd(&npl_s, 1u);
      if (li < K1C_PL) {
        pl_s[li] = pslot;
      } else {
        const uint32_t gi = atomicAdd(&wb.npairs[f], 1u);
        if (gi < (uint32_t)wb.PMAX) wb.plist[(size_t)f * wb.PMAX + gi] = pslot;
        else raise_err(err, DERR_FRAME_PAIRS);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S; i += blockDim.x)
    if (vsd_s[i]) atomicAdd(&wb.vs[(size_t)f * wb.SMAX + i], vsd_s[i]);
  const uint32_t m = min(npl_s, K1C_PL);
  if (threadIdx.x == 0) base_s = m ? atomicAdd(&wb.npairs[f], m) : 0u;
  __syncthreads();
  if (base_s + m > (uint32_t)wb.PMAX) {
    if (threadIdx.x == 0) raise_err(err, DERR_FRAME_PAIRS);
  } else {
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) wb.plist[(size_t)f * wb.PMAX + base_s + i] = pl_s[i];
  }
}

__global__ void k_nsmid(int* out) {
  uint32_t n;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
  *out = (int)n;
}
int k1_nsmid() {
  int* d = nullptr;
  int h = 0;
  if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 256;
  k_nsmid<<<1, 1>>>(d);
  if (cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess || h <= 0) h = 256;
  cudaFree(d);
  return h;
}

// ------------------------------------------------------------------------------------------
// K2: pair records (key, s, frame-key slot) for stage 2; detection key-space AABBs;
// S_angle terms max(0, -r_v . n_v) (Eq.3, R21) in semantic mode.  Clears the pair table.
// ------------------------------------------------------------------------------------------
constexpr int K2_THREADS = 256;

template <bool SEM>
__global__ void __launch_bounds__(K2_THREADS) k_pairs(WinDesc wd, WinBufs wb, Params P, int* err, int abl) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int S = F.S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* ab_s = (int32_t*)smem_raw;            // [S][6]
  for (int s = threadIdx.x; s < S; s += blockDim.x)
    for (int k = 0; k < 3; ++k) { ab_s[6 * s + k] = INT32_MAX; ab_s[6 * s + 3 + k] = INT32_MIN; }
  __syncthreads();
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX;
  uint32_t* ptab = wb.ptab + (size_t)f * wb.PC;
  const unsigned long long* ktab = wb.ktab + (size_t)f * wb.PC;
  NSum* nsum = wb.nsum + (size_t)f * wb.PC;
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < np; base += stride) {
    const uint32_t idx = base + lane;
    uint32_t sv = 0xFFFFFFFFu;   // this lane's detection when it has an S_angle term
    float term = 0.f;
    if (idx < np) {
      const uint32_t ps = wb.plist[fo + idx];
      const uint32_t code = ps < (uint32_t)wb.PC ? ptab[ps] : U32_EMPTY;
      const uint32_t s = code >> 24, ks = code & 0xFFFFFFu;
      if (code == U32_EMPTY || s >= (uint32_t)S || ks >= (uint32_t)wb.PC) {
        atomicCAS(err, 0, 1000 + __LINE__);
      } else {
        const uint64_t key = ktab[ks];
        wb.pkey[fo + idx] = key;
        wb.pinfo[fo + idx] = s;
        wb.pfk[fo + idx] = ks;
        ptab[ps] = U32_EMPTY;   // release the pair-table cell for the next window
        int k3[3];
        unpack_key(key, k3[0], k3[1], k3[2]);
        if (!(abl & 2))
          for (int a = 0; a < 3; ++a) {
            atomicMin(&ab_s[6 * s + a], k3[a]);
            atomicMax(&ab_s[6 * s + 3 + a], k3[a]);
          }
        if (SEM && !(abl & 1)) {
          const float n0 = (float)((double)__ldcg(&nsum[ps].x) / NSCALE);
          const float n1 = (float)((double)__ldcg(&nsum[ps].y) / NSCALE);
          const float n2 = (float)((double)__ldcg(&nsum[ps].z) / NSCALE);
          const float nl = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
          if (nl > 0.f) {
            const float r0 = ((float)k3[0] + 0.5f) * P.r - F.pose[3];
            const float r1 = ((float)k3[1] + 0.5f) * P.r - F.pose[7];
            const float r2 = ((float)k3[2] + 0.5f) * P.r - F.pose[11];
            const float rl = sqrtf(r0 * r0 + r1 * r1 + r2 * r2);
            if (rl > 0.f) {
              const float dot = (r0 * n0 + r1 * n1 + r2 * n2) / (rl * nl);
              term = fmaxf(0.f, -dot);
              sv = s;
            }
          }
        }
      }
    }
    if (SEM && !(abl & 16)) {   // S_angle sums: warp sums per distinct detection, one native RED each
      unsigned pending = __ballot_sync(0xffffffffu, sv != 0xFFFFFFFFu);
      while (pending) {
        const int leader = __ffs(pending) - 1;
        const uint32_t s0 = __shfl_sync(0xffffffffu, sv, leader);
        const bool in = sv == s0;
        // fixed point before any sum: the result does not depend on which warp a term lands in
        unsigned long long v = in ? (unsigned long long)llrint((double)term * ANG_SCALE) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const unsigned inb = __ballot_sync(0xffffffffu, in);
        if (lane == leader) {
          const size_t gi = (size_t)f * wb.SMAX + s0;
          atomicAdd(&wb.ang64[gi], v);
          atomicAdd(&wb.ang_cnt[gi], (uint32_t)__popc(inb));
        }
        pending &= ~inb;
      }
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < S && !(abl & 4); s += blockDim.x) {
    const size_t gi = (size_t)f * wb.SMAX + s;
    if (ab_s[6 * s] != INT32_MAX) {
      for (int a = 0; a < 3; ++a) {
        atomicMin(&wb.daabb[6 * gi + a], ab_s[6 * s + a]);
        atomicMax(&wb.daabb[6 * gi + 3 + a], ab_s[6 * s + 3 + a]);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// K3: Eq.1 inputs.  fbar = mean_p f_p (fp64 partial sums, fixed-order reduction) and
// r_p = |f_p - fbar| (fp32, one warp per patch).  rbar and D_p = r_p / (rbar + eps) are
// formed by k_dmap (fixed-order reduction, one CTA per frame).
// ------------------------------------------------------------------------------------------
constexpr int K3_ROWS = 64;

__global__ void __launch_bounds__(256) k_fbar_part(WinDesc wd, WinBufs wb, int Df, int f0, int evict_last) {
  const int f = f0 + blockIdx.y;   // frames [f0, f0 + gridDim.y): one L2-sized group (launch_stage1)
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  if (!F.feats) return;
  const int P = F.Hp * F.Wp;
  const int ch = blockIdx.x;
  const int p0 = ch * K3_ROWS;
  if (p0 >= P) return;
  const int p1 = min(P, p0 + K3_ROWS);
  double* part = wb.fpart + ((size_t)f * wb.FCHUNKS + ch) * Df;
  const uint64_t pol = evict_last ? policy_evict_last() : policy_evict_first();   // grouped: kept for k_poolr
  float xm = 0.f;
  for (int d4 = threadIdx.x; d4 < Df / 4; d4 += blockDim.x) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int p = p0; p < p1; ++p) {
      const float4 x = ld_f4_ef((const float4*)(F.feats + (size_t)p * Df) + d4, pol);
      a0 += x.x; a1 += x.y; a2 += x.z; a3 += x.w;
      xm = fmaxf(xm, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
    }
    part[4 * d4 + 0] = a0; part[4 * d4 + 1] = a1; part[4 * d4 + 2] = a2; part[4 * d4 + 3] = a3;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  if ((threadIdx.x & 31) == 0 && xm > 0.f) atomicMax((int*)&wb.xmax[f], __float_as_int(xm));   // (>= 0: int order)
}

__global__ void __launch_bounds__(256) k_fbar(WinDesc wd, WinBufs wb, int Df, int f0) {
  const int f = f0 + blockIdx.y;
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

// ------------------------------------------------------------------------------------------
// K3d: D_p = r_p / (rbar + eps) in place (Eq.1), one CTA per frame, fixed-order reduction.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_dmap(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.x;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  if (!F.feats) return;
  const int Pn = F.Hp * F.Wp;
  float* rp = wb.rp + (size_t)f * wb.PMAXP;
  __shared__ double red[40];
  double a = 0;
  for (int p = threadIdx.x; p < Pn; p += blockDim.x) a += (double)rp[p];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) red[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    red[32] = t / (double)Pn;   // rbar
    wb.rbar[f] = red[32];
  }
  __syncthreads();
  const double inv = 1.0 / (red[32] + (double)P.eps);
  for (int p = threadIdx.x; p < Pn; p += blockDim.x) rp[p] = (float)((double)rp[p] * inv);
}

// ------------------------------------------------------------------------------------------
// K4: per-detection features, split for balance (a wall-sized mask no longer serialises ~1000
// patches in one CTA):
//  k_filter   (mask, frame): |M_s| from the per-patch counts, mask filter (A1/R8), no-depth
//             drop; semantic: weight sums -> fallback mode (R18), D̄_s (R19)
//  k_pool     (CTA group, mask, frame): D-weighted pooling y_s += w_p f_p and tracking
//             u_s += cnt_sp g_p (R15) over an interleaved share of the bbox patches; per-CTA
//             fixed-order partials reduced into per-mask accumulators (fp32 / fp64 RED)
//  k_finalize (mask, frame): e_s = y/|y| ("nofeat" if 0), S_size, S_angle, S_sem, S_dist, Q
//             (Eq.2-3); t_s = u / sqrt(dot_pin(u, u)) (R15)
// ------------------------------------------------------------------------------------------
constexpr int K4_THREADS = 256;
constexpr int K4_WARPS = K4_THREADS / 32;
constexpr int K4_CTAS = 8;        // CTAs per mask in k_pool

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

struct BoxPatches {   // the patch range of a mask's bbox (every patch with cnt > 0 lies in it)
  int pr0, pc0, npr, npc, n;
  __device__ BoxPatches(const WinBufs& wb, size_t gi, int H, int W, int Hp, int Wp) {
    const int umin = wb.bbox[4 * gi + 0], vmin = wb.bbox[4 * gi + 1];
    const int umax = wb.bbox[4 * gi + 2], vmax = wb.bbox[4 * gi + 3];
    pr0 = pc0 = 0; npr = npc = 0;
    if (umax >= 0) {
      pr0 = (int)((int64_t)vmin * Hp / H);
      pc0 = (int)((int64_t)umin * Wp / W);
      npr = (int)((int64_t)vmax * Hp / H) - pr0 + 1;
      npc = (int)((int64_t)umax * Wp / W) - pc0 + 1;
    }
    n = npr * npc;
  }
  __device__ int patch(int k, int Wp) const { return (pr0 + k / npc) * Wp + pc0 + k % npc; }
  __device__ double npix(int k, int H, int W, int Hp, int Wp) const {   // pixels of patch k (R17)
    const int i = pr0 + k / npc, j = pc0 + k % npc;
    const int64_t rows = ((int64_t)(i + 1) * H + Hp - 1) / Hp - ((int64_t)i * H + Hp - 1) / Hp;
    const int64_t cols = ((int64_t)(j + 1) * W + Wp - 1) / Wp - ((int64_t)j * W + Wp - 1) / Wp;
    return (double)(rows * cols);
  }
};

template <bool SEM>
__global__ void __launch_bounds__(K4_THREADS) k_filter(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int s = blockIdx.x;
  if (s >= F.S) return;
  const int H = F.H, W = F.W, Hp = F.Hp, Wp = F.Wp;
  const size_t gi = (size_t)f * wb.SMAX + s;
  __shared__ double red[40];
  const BoxPatches B(wb, gi, H, W, Hp, Wp);
  const uint32_t* cnt = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP + (size_t)s * wb.PMAXP;
  double asum = 0;
  for (int k = threadIdx.x; k < B.n; k += blockDim.x) asum += (double)cnt[B.patch(k, Wp)];
  const uint32_t area = (uint32_t)block_sum_d(asum, red);
  // A1 mask filter (R8, R28): first failing reason wins: area==0, conf, aspect, area
  const float conf = F.conf ? F.conf[s] : 1.0f;
  int status = 0;
  if (area == 0) status = 1;
  else if (conf < P.min_conf) status = 2;
  else {
    const int64_t bw = (int64_t)wb.bbox[4 * gi + 2] - wb.bbox[4 * gi + 0] + 1;
    const int64_t bh = (int64_t)wb.bbox[4 * gi + 3] - wb.bbox[4 * gi + 1] + 1;
    const int64_t lo = min(bw, bh), hi = max(bw, bh);
    if ((double)hi > (double)P.max_aspect * (double)lo) status = 3;
    else if ((int64_t)area < (int64_t)P.min_area) status = 1;
    else if (wb.vs[gi] == 0) status = 4;            // O3 no valid depth
  }
  float* qf = wb.qf + 6 * gi;
  if (threadIdx.x == 0) {
    wb.area[gi] = area;
    wb.status[gi] = status;
    wb.pmode[gi] = 0;
    if (status != 0) {
      for (int k = 0; k < 6; ++k) qf[k] = k == 4 ? -1.f : 0.f;
      wb.tok[gi] = 0;
    }
  }

}

// ------------------------------------------------------------------------------------------
// K4b k_poolr: one pass over the frame's patch tokens.  A warp owns a segment of up to
// K4R_SEG patches of one patch row; for each patch it reads the CLIP row once, forms
// r_p = |f_p - fbar| (Eq.1 numerator, written for k_dmap) and, for every kept mask covering the
// patch, adds r_p cover f_p to the mask's pooled sum (P:128 with D_p = r_p / (rbar + eps): the
// common factor 1 / (rbar + eps) cancels in e_s = y / |y| and in the all-zero test of R18) and
// cnt g_p to the tracking sum u_s (R15), plus the scalar sums of R18 / R19.  The warp keeps one
// mask's running sums in its shared-memory slice and flushes them with native REDs when the
// segment moves on to another mask; the other masks of a boundary patch are reduced directly.
// ------------------------------------------------------------------------------------------
constexpr int K4R_SEG = 8;        // patches per warp segment
constexpr int K4R_WARPS = 4;

__device__ __forceinline__ void red_add4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// bulk asynchronous copies (TMA engine, 1-D) into shared memory, completion on an mbarrier
__device__ __forceinline__ uint32_t sm_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm_addr(dst)),
               "l"(src), "r"(bytes), "r"(sm_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          sm_addr(bar)),
      "r"(parity)
      : "memory");
}

// shared bytes of k_poolr: fbar, the warps' running sums, and (bulk path) two row stages per warp
size_t k4r_smem_bytes(int Df, int Dt, bool bulk) {
  return (size_t)(1 + K4R_WARPS) * Df * 4 + (size_t)K4R_WARPS * Dt * 8 +
         (bulk ? (size_t)K4R_WARPS * 2 * ((size_t)Df * 4 + (size_t)Dt * 2) : 0);
}

#ifndef K4R_MINB
#define K4R_MINB 4
#endif
// BULK: a warp's patch rows (CLIP row + tracking row) arrive by bulk async copies into a
// two-stage shared-memory ring, the next patch in flight while this one is reduced.
template <bool SEM, bool BULK>
__global__ void __launch_bounds__(K4R_WARPS * 32, K4R_MINB) k_poolr(WinDesc wd, WinBufs wb, Params P, int f0) {
  const int f = f0 + blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int H = F.H, W = F.W, Hp = F.Hp, Wp = F.Wp, S = F.S, Df = P.Df, Dt = P.Dt;
  const bool pool = SEM && F.feats;
  if (!pool && Dt == 0) return;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int segs_row = (Wp + K4R_SEG - 1) / K4R_SEG;
  const int seg = blockIdx.x * K4R_WARPS + warp;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* fb_s = (float*)smem_raw;                                       // [Df] fbar
  float* ya = fb_s + Df + (size_t)warp * Df;                            // [Df] running pooled sum
  double* ua = (double*)(fb_s + (size_t)(1 + K4R_WARPS) * Df) + (size_t)warp * Dt;   // [Dt]
  // (BULK) the warp's two stages: CLIP row [Df] floats, then tracking row [Dt] bf16
  unsigned char* stg = (unsigned char*)((double*)(fb_s + (size_t)(1 + K4R_WARPS) * Df) + (size_t)K4R_WARPS * Dt) +
                       (size_t)warp * 2 * ((size_t)Df * 4 + (size_t)Dt * 2);
  __shared__ __align__(8) uint64_t bar_s[K4R_WARPS][2];
  if (pool)
    for (int d = threadIdx.x; d < Df; d += blockDim.x) fb_s[d] = wb.fbar[(size_t)f * Df + d];
  for (int d = lane; d < Df; d += 32) ya[d] = 0.f;
  for (int d = lane; d < Dt; d += 32) ua[d] = 0.0;
  __syncthreads();
  if (seg >= Hp * segs_row) return;
  const int pr = seg / segs_row, pc0 = (seg - pr * segs_row) * K4R_SEG, pc1 = min(Wp, pc0 + K4R_SEG);
  const size_t gbase = (size_t)f * wb.SMAX;
  const uint32_t* cnt = wb.cnt + gbase * wb.PMAXP;
  const int D4 = Df / 4, nq4 = (D4 + 31) / 32;
  const int nch = (S + 31) >> 5;   // <= 8 (S <= 255)
  const bool tvec = (Dt & 3) == 0;   // tracking rows as uint2 (4 bf16) per lane (Dt <= 512)
  // this lane's kept flags (status 0) for masks lane, lane + 32, ... (S <= 255)
  uint32_t keptl = 0;
  for (int q = 0; q < nch; ++q)
    if (32 * q + lane < S && wb.status[gbase + 32 * q + lane] == 0) keptl |= 1u << q;
  const int rows = ((pr + 1) * H + Hp - 1) / Hp - (pr * H + Hp - 1) / Hp;
  int cur = -1;                     // mask whose sums the warp's slice holds
  double sc0 = 0, sc1 = 0, sc2 = 0; // its R18 / R19 scalar sums
  bool scw = false;                 // some weight > 0 (R18)
  const float xmx = pool ? __ldcg(&wb.xmax[f]) : 0.f;
  const double se = ldexp(1.0, pool_scale_exp(Hp * Wp, Df, xmx, false));   // fixed-point scales (exact)
  const double sp = ldexp(1.0, pool_scale_exp(Hp * Wp, Df, xmx, true));
  auto fx = [&](float v) { return (unsigned long long)llrint((double)v * se); };
  auto fxp = [&](double v) { return (unsigned long long)llrint(v * sp); };
  auto flush = [&]() {
    if (cur < 0) return;
    const size_t gi = gbase + cur;
    if (pool) {
      unsigned long long* y = (unsigned long long*)(wb.emb64 + gi * Df);
      for (int d4 = lane; d4 < D4; d4 += 32) {
        const float4 a = ((float4*)ya)[d4];
        atomicAdd(&y[4 * d4 + 0], fx(a.x)); atomicAdd(&y[4 * d4 + 1], fx(a.y));
        atomicAdd(&y[4 * d4 + 2], fx(a.z)); atomicAdd(&y[4 * d4 + 3], fx(a.w));
        ((float4*)ya)[d4] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) {
        unsigned long long* ps = (unsigned long long*)(wb.psum64 + gi * 3);
        atomicAdd(&ps[0], fxp(sc0));
        atomicAdd(&ps[1], fxp(sc1));
        atomicAdd(&ps[2], fxp(sc2));
        if (scw) wb.pw[gi] = 1u;
      }
    }
    scw = false;
    double* u = wb.trk + gi * Dt;
    for (int d = lane; d < Dt; d += 32) {
      if (ua[d] != 0.0) atomicAdd(&u[d], ua[d]);
      ua[d] = 0.0;
    }
    sc0 = sc1 = sc2 = 0;
    cur = -1;
    __syncwarp();
  };
  auto prefetch = [&](int pp) {   // the next patch's rows into L2 (one 128-byte line per lane)
    if (pool && lane * 32 < Df) asm volatile("prefetch.global.L2 [%0];" ::"l"(F.feats + (size_t)pp * Df + lane * 32));
    if (Dt > 0 && lane * 64 < Dt) asm volatile("prefetch.global.L2 [%0];" ::"l"(F.track + (size_t)pp * Dt + lane * 64));
  };
  const uint32_t stage_bytes = (uint32_t)Df * 4 + (uint32_t)Dt * 2;
  auto issue = [&](int pcx) {   // lane 0: the rows of patch pcx into stage (pcx - pc0) & 1
    const int st = (pcx - pc0) & 1, pp = pr * Wp + pcx;
    unsigned char* b = stg + (size_t)st * stage_bytes;
    const uint32_t fb = pool ? (uint32_t)Df * 4 : 0u, tb = (uint32_t)Dt * 2;
    mbar_expect_tx(&bar_s[warp][st], fb + tb);
    if (fb) bulk_g2s(b, F.feats + (size_t)pp * Df, fb, &bar_s[warp][st]);
    if (tb) bulk_g2s(b + (size_t)Df * 4, F.track + (size_t)pp * Dt, tb, &bar_s[warp][st]);
  };
  if (BULK) {
    if (lane == 0) {
      mbar_init(&bar_s[warp][0], 1);
      mbar_init(&bar_s[warp][1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      issue(pc0);
      if (pc0 + 1 < pc1) issue(pc0 + 1);
    }
    __syncwarp();
  } else {
    prefetch(pr * Wp + pc0);
  }
  for (int pcx = pc0; pcx < pc1; ++pcx) {
    const int p = pr * Wp + pcx;
    const int st = (pcx - pc0) & 1;
    if (BULK) mbar_wait(&bar_s[warp][st], ((pcx - pc0) >> 1) & 1);
    else if (pcx + 1 < pc1) prefetch(p + 1);
    const float4* srow = (const float4*)(stg + (size_t)st * stage_bytes);
    const uint2* strk = (const uint2*)(stg + (size_t)st * stage_bytes + (size_t)Df * 4);
    float4 x[8];
    float r = 0.f;
    if (pool) {   // the patch's CLIP row and r_p (k_resid's arithmetic: per-lane fmaf, xor butterfly)
      const float4* row = BULK ? srow : (const float4*)(F.feats + (size_t)p * Df);
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < nq4 && lane + 32 * i < D4) {
          x[i] = BULK ? row[lane + 32 * i] : ld_f4_ef(row + lane + 32 * i, pol);
          const float4 m = ((const float4*)fb_s)[lane + 32 * i];
          const float a = x[i].x - m.x, b = x[i].y - m.y, c = x[i].z - m.z, e = x[i].w - m.w;
          acc = fmaf(a, a, acc); acc = fmaf(b, b, acc); acc = fmaf(c, c, acc); acc = fmaf(e, e, acc);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      r = sqrtf(acc);
      if (lane == 0) wb.rp[(size_t)f * wb.PMAXP + p] = r;
    }
    // the patch's tracking row, once: lane l holds elements 4 l + j + 128 k (uint2 = 4 bf16)
    uint2 gv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      gv[k] = make_uint2(0u, 0u);
      if (tvec && 4 * lane + 128 * k < Dt)
        gv[k] = BULK ? strk[lane + 32 * k] : __ldcs((const uint2*)(F.track + (size_t)p * Dt) + lane + 32 * k);
    }
    // keep the slice's mask if it covers p, else flush it: p's first mask takes the slice
    if (cur >= 0 && cnt[(size_t)cur * wb.PMAXP + p] == 0) flush();
    // patch pixel count (R17), 32-bit: W, H <= 16384
    const int cols = ((pcx + 1) * W + Wp - 1) / Wp - (pcx * W + Wp - 1) / Wp;
    const double npix = (double)(rows * cols);
    for (int q = 0; q < nch; ++q) {   // the kept masks covering p, 32 per ballot
      const uint32_t c_l = ((keptl >> q) & 1u) ? cnt[(size_t)(32 * q + lane) * wb.PMAXP + p] : 0u;
      for (uint32_t todo = __ballot_sync(0xffffffffu, c_l != 0); todo;) {
        const int b = __ffs(todo) - 1;
        todo &= todo - 1;
        const int s = 32 * q + b;
        const uint32_t c = __shfl_sync(0xffffffffu, c_l, b);
        if (cur < 0) cur = s;
        const double cov = (double)c / npix;
        const bool use = (double)c >= (double)P.cover_min * npix;   // R17, exact
        const float w = (float)((double)r * cov);
        const uint16_t* g = F.track + (size_t)p * Dt;
        if (s == cur) {
          if (pool) {
            if (use) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (i < nq4 && lane + 32 * i < D4) {
                  float4 a = ((float4*)ya)[lane + 32 * i];
                  a.x = fmaf(w, x[i].x, a.x); a.y = fmaf(w, x[i].y, a.y);
                  a.z = fmaf(w, x[i].z, a.z); a.w = fmaf(w, x[i].w, a.w);
                  ((float4*)ya)[lane + 32 * i] = a;
                }
              }
              sc0 += (double)r * cov;
              scw = scw || (r > 0.f && cov > 0.0);
            }
            sc1 += cov * (double)r;
            sc2 += cov;
          }
          if (tvec) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int d0 = 4 * lane + 128 * k;
              if (d0 < Dt) {
                const uint32_t e[4] = {gv[k].x << 16, gv[k].x & 0xFFFF0000u, gv[k].y << 16, gv[k].y & 0xFFFF0000u};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                  ua[d0 + jj] = __dadd_rn(ua[d0 + jj], __dmul_rn((double)c, (double)__uint_as_float(e[jj])));
              }
            }
          } else {
            for (int d = lane; d < Dt; d += 32)
              ua[d] = __dadd_rn(ua[d], __dmul_rn((double)c, (double)__uint_as_float((uint32_t)g[d] << 16)));
          }
        } else {   // another mask of a boundary patch: reduce straight into its sums
          const size_t gi = gbase + s;
          if (pool) {
            if (use) {
              unsigned long long* y = (unsigned long long*)(wb.emb64 + gi * Df);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (i < nq4 && lane + 32 * i < D4) {
                  const int d = 4 * (lane + 32 * i);
                  atomicAdd(&y[d + 0], fx(w * x[i].x)); atomicAdd(&y[d + 1], fx(w * x[i].y));
                  atomicAdd(&y[d + 2], fx(w * x[i].z)); atomicAdd(&y[d + 3], fx(w * x[i].w));
                }
            }
            if (lane == 0) {
              unsigned long long* ps = (unsigned long long*)(wb.psum64 + gi * 3);
              if (use) {
                atomicAdd(&ps[0], fxp((double)r * cov));
                if (r > 0.f && cov > 0.0) wb.pw[gi] = 1u;
              }
              atomicAdd(&ps[1], fxp(cov * (double)r));
              atomicAdd(&ps[2], fxp(cov));
            }
          }
          double* u = wb.trk + gi * Dt;
          if (tvec) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int d0 = 4 * lane + 128 * k;
              if (d0 < Dt) {
                const uint32_t e[4] = {gv[k].x << 16, gv[k].x & 0xFFFF0000u, gv[k].y << 16, gv[k].y & 0xFFFF0000u};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                  atomicAdd(&u[d0 + jj], __dmul_rn((double)c, (double)__uint_as_float(e[jj])));
              }
            }
          } else {
            for (int d = lane; d < Dt; d += 32)
              atomicAdd(&u[d], __dmul_rn((double)c, (double)__uint_as_float((uint32_t)g[d] << 16)));
          }
        }
      }
    }
    if (BULK) {   // the stage is free again: the patch after next goes into it
      __syncwarp();
      if (lane == 0 && pcx + 2 < pc1) issue(pcx + 2);
    }
  }
  flush();
}

// R18 fallback: a kept mask whose weights are all zero is pooled unweighted over its patches
// with cnt > 0 (its weighted sum is exactly zero).  Rare; CTAs of other masks exit at once.
template <bool SEM>
__global__ void __launch_bounds__(K4_THREADS) k_fallback(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.z;
  if (!SEM || f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int s = blockIdx.y;
  if (s >= F.S || !F.feats) return;
  const size_t gi = (size_t)f * wb.SMAX + s;
  if (wb.status[gi] != 0 || wb.pw[gi]) return;
  const int H = F.H, W = F.W, Hp = F.Hp, Wp = F.Wp, Df = P.Df;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const BoxPatches B(wb, gi, H, W, Hp, Wp);
  const int stride = K4_CTAS * K4_WARPS;
  const uint32_t* cnt = wb.cnt + (size_t)f * wb.SMAX * wb.PMAXP + (size_t)s * wb.PMAXP;
  unsigned long long* y = (unsigned long long*)(wb.emb64 + gi * Df);
  const double se = ldexp(1.0, pool_scale_exp(Hp * Wp, Df, __ldcg(&wb.xmax[f]), false));
  for (int k = blockIdx.x * K4_WARPS + warp; k < B.n; k += stride) {
    const int p = B.patch(k, Wp);
    if (!cnt[p]) continue;
    const float* row = F.feats + (size_t)p * Df;
    for (int d = lane; d < Df; d += 32) atomicAdd(&y[d], (unsigned long long)llrint((double)row[d] * se));
  }
}

template <bool SEM>
__global__ void __launch_bounds__(K4_THREADS) k_finalize(WinDesc wd, WinBufs wb, Params P) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const FrameDesc& F = wd.f[f];
  const int s = blockIdx.x;
  if (s >= F.S) return;
  const size_t gi = (size_t)f * wb.SMAX + s;
  if (wb.status[gi] != 0) return;
  const int H = F.H, W = F.W, Df = P.Df, Dt = P.Dt;
  __shared__ double red[40];
  float* qf = wb.qf + 6 * gi;
  if (SEM && F.feats) {
    float* emb = wb.emb + gi * Df;
    const long long* y64 = wb.emb64 + gi * Df;
    const double sinv = ldexp(1.0, -pool_scale_exp(F.Hp * F.Wp, Df, wb.xmax[f], false));
    double yy = 0;
    for (int d = threadIdx.x; d < Df; d += blockDim.x) {
      const double y = (double)y64[d] * sinv;
      yy += y * y;
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
    const double rn = 1.0 / sqrt(yy);
    double eg = 0, gg = 0;
    for (int d = threadIdx.x; d < Df; d += blockDim.x) {
      const float e = (float)((double)y64[d] * sinv * rn);
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
      const double s_size = fmin((double)P.lambda * (double)wb.area[gi] / ((double)H * (double)W), 1.0);
      const uint32_t ac = wb.ang_cnt[gi];
      const double s_angle = ac ? (double)wb.ang64[gi] / ANG_SCALE / (double)ac : 0.0;
      double s_sem = 1.0;
      if (F.gemb) s_sem = gg > 0 ? fmin(fmax(eg / sqrt(gg), 0.0), 1.0) : 0.0;
      // R19: D-bar = sum(cover D) / sum(cover) with D = r / (rbar + eps)
      const long long* ps = wb.psum64 + gi * 3;   // (both scaled by 2^kp: the ratio is unchanged)
      const double dbar = ps[2] > 0 ? (double)ps[1] / (double)ps[2] / (wb.rbar[f] + (double)P.eps) : 0.0;
      qf[5] = (float)dbar;
      wb.pmode[gi] = wb.pw[gi] ? 0 : 1;   // 1: all-zero weights -> unweighted pooling (R18)
      const double s_dist = 0.5 + 0.5 * dbar;
      qf[0] = (float)s_size; qf[1] = (float)s_angle; qf[2] = (float)s_sem; qf[3] = (float)s_dist;
      qf[4] = (float)(((s_size * s_angle) * s_sem) * s_dist);
    }
  } else if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) qf[k] = k == 4 ? -1.f : 0.f;   // geometry-only: no embedding
  }
  if (Dt > 0 && threadIdx.x < 32) {
    double* t = wb.trk + gi * Dt;   // holds u_s; normalised in place
    const double nn = dot_pin_warp(t, t, Dt);
    const bool ok = nn > 0.0;
    const double n = ok ? sqrt(nn) : 1.0;
    for (int d = threadIdx.x; d < Dt; d += 32) t[d] = ok ? __ddiv_rn(t[d], n) : 0.0;
    if (threadIdx.x == 0) wb.tok[gi] = ok ? 1 : 0;
  }
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
// DISC_K1_ABLATE (profiling only; results are wrong when set): 1 skip mask planes, 2 skip
// the walk, 8 skip normals
static int k1_ablate() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DISC_K1_ABLATE");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int k1_tiles(int H, int W, bool sem) {
  const int tw = K1_WARPS * k1_cols_out(sem);
  return ((W + tw - 1) / tw) * ((H + K1_TILE_H - 1) / K1_TILE_H);
}

// Release of the frame tables after use (tables much larger than the frames' pair counts, e.g. H's
// 2^20-slot tables for ~10^5 pairs): the key slot of every pair and (semantic mode) its normal-sum
// slot return to EMPTY / 0, instead of a streaming fill of the whole tables before the next window.
__global__ void __launch_bounds__(256) k_release(WinDesc wd, WinBufs wb, int sem) {
  const int f = blockIdx.y;
  if (f >= wd.n) return;
  const uint32_t np = min(wb.npairs[f], (uint32_t)wb.PMAX);
  const size_t fo = (size_t)f * wb.PMAX, to = (size_t)f * wb.PC;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const uint32_t ks = wb.pfk[fo + i];
    if (ks < (uint32_t)wb.PC) __stcs(&wb.ktab[to + ks], (unsigned long long)KEY_EMPTY);
    if (sem) {
      const uint32_t ps = wb.plist[fo + i];
      if (ps < (uint32_t)wb.PC) wb.nsum[to + ps] = NSum{0, 0, 0, 0};
    }
  }
}

int launch_stage1(const WinDesc& wd, const WinBufs& wb, const Params& P, int* err, bool sem, int maxS,
                  int maxHp, int maxW, int maxWp, int maxP, int rows_cap, int nsm, int nres, cudaStream_t st,
                  cudaEvent_t ev0, cudaEvent_t ev1, bool fill_ktab, bool fill_nsum, bool release) {
  const int n = wd.n;
  (void)rows_cap; (void)maxW;
  int k1_grid = 1;
  for (int i = 0; i < n; ++i) k1_grid = std::max(k1_grid, k1_tiles(wd.f[i].H, wd.f[i].W, sem));
  (void)maxHp; (void)maxWp;
  k_win_init<<<dim3(8, n), 256, 0, st>>>(wd, wb);
  debug_check(st, "k_win_init", -1);
  // per-pair normal sums start from zero and the key tables empty: either one streaming fill per
  // window (tables sized close to the frames' pair counts: scattered zeroing of partial lines costs
  // more) or, when the previous window released its slots (k_release), nothing to do
  int launches = 0;
  if (sem && fill_nsum) { k_fill_cs<<<4 * nsm, 256, 0, st>>>((uint4*)wb.nsum, (size_t)n * wb.PC * 2, 0u); ++launches; }
  if (fill_ktab) { k_fill_cs<<<4 * nsm, 256, 0, st>>>((uint4*)wb.ktab, (size_t)n * wb.PC / 2, 0xFFFFFFFFu); ++launches; }
  if (ev0) cudaEventRecord(ev0, st);
  int64_t maxHW = 1;
  bool vec = true;
  int nbits = 0, nbytes = 0;   // frames with bit-packed / byte mask planes (frames without masks: either)
  for (int i = 0; i < n; ++i) {
    maxHW = std::max(maxHW, (int64_t)wd.f[i].H * wd.f[i].W);
    vec = vec && wd.f[i].vec16;
    if (wd.f[i].S > 0) (wd.f[i].mbits ? nbits : nbytes)++;
  }
  const int items_a = (int)((maxHW + 32 * K1A_SECT - 1) / (32 * K1A_SECT));
  const dim3 ga(K1A_PERSIST * nsm), ba(K1_THREADS);
  const size_t sa = (size_t)maxS * 16;
  if (nbits && nbytes) k_masks<false, 2><<<ga, ba, sa, st>>>(wd, wb, items_a, nres, k1_ablate());
  else if (nbits && vec) k_masks<true, 1><<<ga, ba, sa, st>>>(wd, wb, items_a, nres, k1_ablate());
  else if (nbits) k_masks<false, 1><<<ga, ba, sa, st>>>(wd, wb, items_a, nres, k1_ablate());
  else if (vec) k_masks<true, 0><<<ga, ba, sa, st>>>(wd, wb, items_a, nres, k1_ablate());
  else k_masks<false, 0><<<ga, ba, sa, st>>>(wd, wb, items_a, nres, k1_ablate());
  debug_check(st, "k_masks", -1);
  if (P.db_eps > 0.f) {   // NEXT f3: DBSCAN denoise, then the kept points into the frame tables (k_dbscan.cu)
    launches += launch_dbscan(wd, wb, P, err, sem, nsm, st) - 2;
  } else {
    if (sem) k_walk<true><<<K1B_PERSIST * nsm, K1_THREADS, (size_t)maxS * 4, st>>>(wd, wb, P, err, k1_grid, nres, k1_ablate());
    else k_walk<false><<<K1B_PERSIST * nsm, K1_THREADS, (size_t)maxS * 4, st>>>(wd, wb, P, err, k1_grid, nres, k1_ablate());
    debug_check(st, "k_walk", -1);
    if (sem) k_dedup<true><<<dim3(K1C_BLOCKS, n), 256, (size_t)maxS * 4, st>>>(wd, wb, err);
    else k_dedup<false><<<dim3(K1C_BLOCKS, n), 256, (size_t)maxS * 4, st>>>(wd, wb, err);
    debug_check(st, "k_dedup", -1);
  }
  if (ev1) cudaEventRecord(ev1, st);
  const size_t sm2 = (size_t)maxS * 6 * 4;
  const int g2 = 64;
  static const int k2abl = getenv("DISC_K2_ABLATE") ? atoi(getenv("DISC_K2_ABLATE")) : 0;   // profiling only
  if (sem) k_pairs<true><<<dim3(g2, n), K2_THREADS, sm2, st>>>(wd, wb, P, err, k2abl);
  else k_pairs<false><<<dim3(g2, n), K2_THREADS, sm2, st>>>(wd, wb, P, err, k2abl);
  debug_check(st, "k_pairs", -1);
  if (release) {
    k_release<<<dim3(32, n), 256, 0, st>>>(wd, wb, sem ? 1 : 0);
    debug_check(st, "k_release", -1);
    ++launches;
  }
  int segs = 1;
  for (int i = 0; i < n; ++i)
    segs = std::max(segs, wd.f[i].Hp * ((wd.f[i].Wp + K4R_SEG - 1) / K4R_SEG));
  const int gx = (segs + K4R_WARPS - 1) / K4R_WARPS;
  // bulk path: 16-byte rows (Df % 4 == 0 holds; Dt % 8 == 0) and 16-byte aligned token arrays
  // the bulk-copy variant measured slower (fewer resident warps for its staging rings): opt-in
  static const bool bulk_ok = getenv("DISC_POOLR_BULK") != nullptr;
  bool bulk = bulk_ok && (P.Dt % 8) == 0 && P.Dt <= 512;
  for (int i = 0; i < n && bulk; ++i)
    bulk = (((uintptr_t)wd.f[i].feats | (uintptr_t)wd.f[i].track) & 15) == 0;
  const size_t smr = k4r_smem_bytes(P.Df, P.Dt, bulk);
  static size_t smr_set[2] = {0, 0};
  if (smr != smr_set[bulk]) {
    if (bulk) {
      cudaFuncSetAttribute(k_poolr<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
      cudaFuncSetAttribute(k_poolr<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
    } else {
      cudaFuncSetAttribute(k_poolr<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
      cudaFuncSetAttribute(k_poolr<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
    }
    smr_set[bulk] = smr;
  }
  if (sem) {
    k_filter<true><<<dim3(maxS, n), K4_THREADS, 0, st>>>(wd, wb, P);
    debug_check(st, "k_filter", -1);
    // Eq.1's mean f-bar and the pooling pass read the same CLIP tokens: run them per group of frames
    // whose tokens fit in L2 (<= 48 MB), so the second read hits L2 (first read evict-last, second
    // evict-first) instead of streaming the window's tokens from HBM twice
    // (measured: per-group launches leave the GPU under-filled and serialise -- stage 1 per window
    // +0.26 ms on H, +1 ms on R -- more than the second HBM read costs, so one group by default;
    // DISC_CLIP_GROUP_MB=<L2 budget> enables the grouping)
    const int nch = (maxP + K3_ROWS - 1) / K3_ROWS;
    const int64_t tok_bytes = std::max<int64_t>(1, (int64_t)maxP * P.Df * 4);
    static const int64_t grp_mb = getenv("DISC_CLIP_GROUP_MB") ? atoll(getenv("DISC_CLIP_GROUP_MB")) : 0;
    const int gsz = grp_mb > 0 ? (int)std::max<int64_t>(1, std::min<int64_t>(n, (grp_mb << 20) / tok_bytes)) : n;
    for (int g0 = 0; g0 < n; g0 += gsz) {
      const int gn = std::min(gsz, n - g0);
      k_fbar_part<<<dim3(nch, gn), 256, 0, st>>>(wd, wb, P.Df, g0, gsz < n ? 1 : 0);
      k_fbar<<<dim3((P.Df + 255) / 256, gn), 256, 0, st>>>(wd, wb, P.Df, g0);
      if (bulk) k_poolr<true, true><<<dim3(gx, gn), K4R_WARPS * 32, smr, st>>>(wd, wb, P, g0);
      else k_poolr<true, false><<<dim3(gx, gn), K4R_WARPS * 32, smr, st>>>(wd, wb, P, g0);
      launches += 3;
    }
    debug_check(st, "k_fbar_part / k_fbar / k_poolr", -1);
    k_dmap<<<n, 1024, 0, st>>>(wd, wb, P);
    debug_check(st, "k_dmap", -1);
    k_fallback<true><<<dim3(K4_CTAS, maxS, n), K4_THREADS, 0, st>>>(wd, wb, P);
    debug_check(st, "k_fallback", -1);
    k_finalize<true><<<dim3(maxS, n), K4_THREADS, 0, st>>>(wd, wb, P);
    debug_check(st, "k_finalize", -1);
  } else {
    k_filter<false><<<dim3(maxS, n), K4_THREADS, 0, st>>>(wd, wb, P);
    debug_check(st, "k_filter", -1);
    if (bulk) k_poolr<false, true><<<dim3(gx, n), K4R_WARPS * 32, smr, st>>>(wd, wb, P, 0);
    else k_poolr<false, false><<<dim3(gx, n), K4R_WARPS * 32, smr, st>>>(wd, wb, P, 0);
    debug_check(st, "k_poolr", -1);
    k_finalize<false><<<dim3(maxS, n), K4_THREADS, 0, st>>>(wd, wb, P);
    debug_check(st, "k_finalize", -1);
  }
  return (sem ? 9 : 8) + launches;   // the launches above on s1, counted exactly (bench.py reports them)
}

}  // namespace disc
