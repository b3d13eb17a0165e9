// k_stage1.cuh -- device helpers of stage 1 shared by the mask pass (k_frame.cu) and the DBSCAN
// denoise path (k_dbscan.cu): the pinned R5 world point and key, the frame hash tables, R21 normals.
#pragma once
#include "disc_common.cuh"

namespace disc {

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

// Same result as point_key (floor of the correctly rounded quotient, R5) at a fraction of the
// cost: q = x * fl(1/r) differs from fl(x/r) by at most ~1.8e-7 |q| (two roundings), so whenever
// no integer lies within |q| * 1e-6 of q, floor(q) == floor(fl(x/r)); otherwise fall back to the
// IEEE division.
__device__ __forceinline__ float floor_div_pinned(float x, float r, float rinv) {
  const float q = x * rinv;
  const float fq = floorf(q);
  const float d = q - fq;
  const float tol = fabsf(q) * 1e-6f + 1e-30f;
  if (d > tol && d < 1.0f - tol) return fq;
  return floorf(__fdiv_rn(x, r));
}

__device__ __forceinline__ bool point_key_fast(const float p[3], float r, float rinv, uint64_t& key) {
  int k[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float q = floor_div_pinned(p[i], r, rinv);
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

// native vector float reduction at L2 (fire-and-forget; shared-memory float atomics are CAS loops)
// fixed-point normal sums (NSum): fire-and-forget 64-bit integer reductions
__device__ __forceinline__ void nsum_add_fx(NSum* p, long long a, long long b, long long c) {
  if (a) atomicAdd((unsigned long long*)&p->x, (unsigned long long)a);
  if (b) atomicAdd((unsigned long long*)&p->y, (unsigned long long)b);
  if (c) atomicAdd((unsigned long long*)&p->z, (unsigned long long)c);
}
__device__ __forceinline__ void nsum_add(NSum* p, float a, float b, float c) {
  nsum_add_fx(p, llrint((double)a * NSCALE), llrint((double)b * NSCALE), llrint((double)c * NSCALE));
}
__device__ __forceinline__ void red_add3(float4* p, float a, float b, float c) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(0.f)
               : "memory");
}

// R21: n = (P(u+1,v) - P(u-1,v)) x (P(u,v+1) - P(u,v-1)), oriented so n . (cam - P) >= 0.
__device__ __forceinline__ bool normal_from(const FrameDesc& F, const float pc[3], const float pl[3],
                                            const float pr[3], const float pu[3], const float pd[3], float n[3]) {
  const float a0 = pr[0] - pl[0], a1 = pr[1] - pl[1], a2 = pr[2] - pl[2];
  const float b0 = pd[0] - pu[0], b1 = pd[1] - pu[1], b2 = pd[2] - pu[2];
  n[0] = a1 * b2 - a2 * b1;
  n[1] = a2 * b0 - a0 * b2;
  n[2] = a0 * b1 - a1 * b0;
  if (n[0] == 0.f && n[1] == 0.f && n[2] == 0.f) return false;
  const float o = n[0] * (F.pose[3] - pc[0]) + n[1] * (F.pose[7] - pc[1]) + n[2] * (F.pose[11] - pc[2]);
  if (o < 0.f) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
  return true;
}

}  // namespace disc
