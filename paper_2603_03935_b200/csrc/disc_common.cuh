// disc_common.cuh -- device-side types and helpers shared by libdisc's kernels.
//
// Product code of the CUDA path.  Shares nothing with oracle/ (the CPU checker).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/disc.h"

namespace disc {

constexpr int MAXWIN = 32;
#ifndef K1_PT_SLOTS
#define K1_PT_SLOTS 2048   // a far wall puts ~1000 distinct voxels in one 32x128 tile
#endif
constexpr int K1_PT = K1_PT_SLOTS;         // K1 CTA pair slots (two per CTA key-table slot)
constexpr int K1_SLOTS_PER_SM = 16;    // K1 scratch blocks per SM (>= resident K1 CTAs per SM)
constexpr uint64_t KEY_EMPTY = ~0ull;       // valid packed keys have bit 63 clear (R6)
constexpr uint32_t U32_EMPTY = 0xFFFFFFFFu;
constexpr uint32_t LAB_TOMB = 0xFFFFFFFEu;  // membership label removed by a relabel
constexpr int KEY_BIAS = 1 << 20;           // R6
constexpr int INLINE_LABELS = 5;
constexpr int CHUNK_LABELS = 7;

// error codes raised on the device (sticky; surfaced at synchronising calls)
enum DevErr : int {
  DERR_NONE = 0,
  DERR_FRAME_PAIRS = 1,     // per-frame (s,key) table full
  DERR_MAP_KEYS = 2,        // voxel hash full
  DERR_OVF_POOL = 3,        // overflow label chunks exhausted
  DERR_ARENA = 4,           // per-instance key list arena exhausted
  DERR_TRIPLES = 5,         // per-frame (s,j) count table full
  DERR_INSTANCES = 6,       // max_instances exceeded
  DERR_STAGE = 7,           // per-frame staging list full
  DERR_BOUNDS = 8,          // an index past its array (only raised by a -DDISC_BOUNDS build)
};

// ---- voxel map (stage 2) -------------------------------------------------------------
// One 32-byte slot per voxel key: the key plus the labels (physical instance labels) of
// every instance containing it (the membership relation bucketed by key, R12: instances
// may share voxels).  More than 5 labels spill into 32-byte overflow chunks.
struct __align__(32) KeySlot {
  unsigned long long key;
  uint32_t lab[INLINE_LABELS];
  uint32_t ovf;
};
struct __align__(32) OvfChunk {
  uint32_t lab[CHUNK_LABELS];
  uint32_t next;
};

// A (mask, voxel) pair's sum of pixel normals (R21) in 64-bit fixed point (x 2^40): integer atomics
// are order-independent, so S_angle (and Q) are bit-reproducible whatever the order of the adds
struct __align__(32) NSum {
  long long x, y, z, pad;
};
constexpr double NSCALE = 1099511627776.0;   // 2^40

struct FrameDesc {                // one frame's inputs, passed by value to kernels
  const float* depth;
  const uint8_t* masks;
  const float* conf;
  const float* feats;
  const float* gemb;
  const uint16_t* track;
  const uint32_t* mbits;          // bit-packed masks (disc_frame::mask_bits) or nullptr: `masks`
  float pose[12];                 // rows 0..2 of the camera->world matrix
  float fx, fy, cx, cy;
  int64_t frame_id;
  int32_t H, W, S, Hp, Wp;
  int32_t vec16;                  // vector path: H*W % 32 == 0, masks 32-B and depth 16-B aligned
};

// pixel p (= v*W + u) of mask s, from whichever of the two plane formats the frame carries
__device__ __forceinline__ bool mask_at(const FrameDesc& F, int s, size_t p) {
  if (F.mbits) return (__ldg(F.mbits + (size_t)s * (((size_t)F.H * F.W + 31) >> 5) + (p >> 5)) >> (p & 31)) & 1u;
  return F.masks[(size_t)s * F.H * F.W + p] != 0;
}

struct WinDesc {
  FrameDesc f[MAXWIN];
  int32_t n;
  int32_t Df, Dt;   // feature widths (accumulator zeroing in k_win_init)
};

struct Params {                   // method constants
  float r, tau_geo, tau_vis, dmin, dmax, min_conf, max_aspect, cover_min, lambda, eps;
  int32_t min_area, Df, Dt;
  float db_eps;                   // DBSCAN denoise (R42): 0 = off
  int32_t db_min;
  int32_t refine;                 // f2 active-set refinement (R43): 0 = off
};

// ---- per-window stage-1 buffers (device pointers, strides per frame) -----------------
struct WinBufs {
  unsigned long long* ktab;   // [win][PC] frame key table (packed key)
  uint32_t* ptab;             // [win][PC] frame (s,kslot) pair table (code = s<<24 | kslot)
  NSum* nsum;                 // [win][PC] per-pair normal sums (semantic mode)
  uint32_t* plist;            // [win][PMAX] pair slots in insertion order
  uint32_t* npairs;           // [win]
  // K1b -> K1c: each tile's distinct (s, key) items with their normal sums
  unsigned long long* rkey;   // [win][PMAX] key
  uint32_t* rs;               // [win][PMAX] mask index s
  NSum* rn;                   // [win][PMAX] normal sum (semantic mode)
  uint32_t* rcount;           // [win] records reserved; a tile whose block passes RCAP inserts its
                              // items itself and writes KEY_EMPTY into its records below RCAP
  uint32_t* cnt;              // [win][SMAX][PMAXP] mask pixels per patch
  uint32_t* area;             // [win][SMAX]
  int32_t* bbox;              // [win][SMAX][4] umin, vmin, umax, vmax
  uint32_t* vs;               // [win][SMAX] |V_s|
  int32_t* daabb;             // [win][SMAX][6] key-space aabb of V_s

  uint32_t* ang_cnt;          // [win][SMAX]
  unsigned long long* oor;    // [win] key_out_of_range
  // pair records for stage 2
  unsigned long long* pkey;   // [win][PMAX] key
  uint32_t* pinfo;            // [win][PMAX] mask index s
  uint32_t* pfk;              // [win][PMAX] frame key-table slot
  uint32_t* pms;              // [win][PMAX] map slot found by K5 (or U32_EMPTY)
  uint2* plab;                // [win][PMAX] the slot's first two labels seen by K5 (K7 skips inserts of a present label)
  uint32_t* pnext;            // [win][PMAX] next pair of the frame on the same map slot (speculative counting)
  uint32_t* s2sm;             // [8] (shared by both buffers) SMs hosting a running k_stage2 CTA: bits [0, 5) words,
                              // [5] running k_stage2 CTAs -- stage 1's persistent CTAs keep off exactly those SMs
  // semantic
  double* fpart;              // [win][FCHUNKS][Df] partial column sums
  float* fbar;                // [win][Df]
  float* rp;                  // [win][PMAXP] residual norms r_p (D_p after k_dmap)
  double* rbar;               // [win] mean r_p (Eq.1)
  // Order-independent (bit-reproducible) accumulation: the pooled sums, the R18 / R19 sums and the
  // S_angle sums are 64-bit fixed point (integer atomics are associative), with a per-frame power-of-two
  // scale from the tokens' largest |component| (xmax, k_fbar_part) -- see pool_scale()
  long long* emb64;           // [win][SMAX][Df] pooled sum y_s x 2^ke
  long long* psum64;          // [win][SMAX][3] R18 / R19 sums (with r_p for D_p) x 2^kp: weight, cover r, cover
  unsigned long long* ang64;  // [win][SMAX] S_angle term sum x 2^40
  uint32_t* pw;               // [win][SMAX] 1: some weight > 0 (R18: else unweighted pooling)
  float* xmax;                // [win] max |token component| of the frame
  int32_t* status;            // [win][SMAX]
  float* qf;                  // [win][SMAX][6] s_size, s_angle, s_sem, s_dist, q, dbar
  float* emb;                 // [win][SMAX][Df]
  double* trk;                // [win][SMAX][Dt]  t_s
  uint8_t* tok;               // [win][SMAX] t_s defined (nonzero norm)
  uint8_t* pmode;             // [win][SMAX] 1: unweighted pooling fallback (R18)
  // K1 per-CTA normal-sum scratch: one K1_PT-slot block per resident K1 CTA, acquired per SM
  NSum* k1scr;                // [nsmid][K1_SLOTS_PER_SM][K1_PT], all-zero between CTAs
  uint32_t* k1slot;           // [nsmid] bitmask of the SM's blocks in use
  uint32_t* k1ctr;            // [2] K1a / K1b work-item counters (zeroed by K0)
  uint16_t* m0map;            // [win][MPIX] per pixel: first mask (low byte, 0xFF none), bit 8 = in a
                              // second mask (R9); written by K1a
  int64_t MPIX;
  uint32_t* s2bar;            // [1] stage-2 grid barrier counter (zeroed by K0)
  int32_t PC;                 // frame table capacity (power of 2)
  int32_t PMAX, SMAX, PMAXP, FCHUNKS;
  int32_t RCAP;               // record list capacity per frame (PMAX; DISC_K1_RCAP lowers it in tests)
  // DBSCAN denoise (R42; allocated when dbscan_eps > 0): each frame's (mask, point) records
  unsigned long long* dbk;    // [win][DBP] sort key: s << 56 | grid cell (3 x 18 bits)
  uint32_t* dbv;              // [win][DBP] pixel index
  unsigned long long* dbk2;   // [win][DBP] sorted keys
  uint32_t* dbv2;             // [win][DBP] sorted pixel indices
  float4* dbx;                // [win][DBP] world point of sorted position (w: pixel index bits)
  uint32_t* dbpar;            // [win][DBP] union-find parent (sorted positions)
  uint32_t* dblab;            // [win][DBP] cluster root position of a point, U32_EMPTY = noise
  uint32_t* dbsz;             // [win][DBP] cluster sizes (at root positions)
  uint8_t* dbcore;            // [win][DBP]
  unsigned long long* dbbest; // [win][SMAX] (size << 32 | ~root pixel) of the kept cluster
  uint32_t* dbn;              // [win] points per frame
  int* dbbeg;                 // [win] segment offsets for the sort
  int* dbend;
  void* dbtmp;                // CUB temporary storage
  size_t dbtmp_bytes;
  int32_t DBP;                // points per frame capacity
};

// ---- map state ---------------------------------------------------------------------------
struct MapState {
  KeySlot* slots;             // [MC]
  unsigned long long* slh;    // [MC] (tag << 32 | first pair) of the speculatively counted frame tagged `tag` on
                              // this slot (wb.pnext chains its other pairs); other tags: none
  OvfChunk* ovf;              // [OVFCAP]
  uint32_t* ovf_top;
  uint32_t OVFCAP;
  uint64_t MC;                // power of two
  // instance table, indexed by id (ids and physical labels share the id space)
  uint8_t* alive;
  uint32_t* phys_of;          // id -> physical label of its memberships
  uint32_t* id_of;            // physical label -> live id
  int64_t* vcount;
  int32_t* obs;
  int64_t* last_seen;
  int32_t* aabb;              // [6]
  float* q;
  float* E;                   // [Df]
  double* T;                  // [Dt]
  double* TT;                 // dot_pin(T_j, T_j) (R15), refreshed whenever T_j changes
  // per physical label key-slot lists (for relabel enumeration)
  unsigned long long* lst_off;
  uint32_t* lst_len;
  uint32_t* lst_cap;
  uint32_t* arena;
  unsigned long long* arena_top;
  unsigned long long ARENA;
  int32_t IMAX;
  uint32_t* stamp;            // [IMAX] K6 generation stamps (instance -> local node id)
  int32_t* local;             // [IMAX]
  int64_t* counters;          // [8]: 0 next_id, 1 live_instances, 2 live_memberships, 3 frame gen
  int* err;
};

// per-frame stage-2 scratch
struct FrameScratch {
  unsigned long long* ctab_key;  // [CC] (s<<32 | j) count table
  uint32_t* ctab_cnt;            // [CC]
  uint32_t* ctab_idx;            // [CC] triple index
  uint32_t* ntrip;               // [1]
  uint8_t* trip_gate;            // [TCAP] visual gate of each triple (R15), computed by CTAs 1.. of stage 2
  uint32_t* gate_done;           // [1] triples gated so far this frame (reset by the association)
  uint32_t* trip_s;              // [TCAP]
  uint32_t* trip_j;
  uint32_t* trip_c;
  uint8_t* trip_edge;
  uint32_t* trip_sd;             // [TCAP] debug export of the association's triples (s, id; trip_c, trip_edge)
  uint32_t* trip_jd;
  // the second count table (speculative counting: frame f+1 is counted while frame f is associated);
  // frame f of a launch uses table (f - f0) & 1, ct2 holds table 1's pointers
  unsigned long long* ctab_key2;
  uint32_t *ctab_cnt2, *ctab_idx2, *ntrip2, *trip_s2, *trip_j2;
  int32_t CC, TCAP;               // count-table slots (power of 2, >= 2 TCAP); triple capacity per frame
  int32_t TCS;                     // triples the association holds in shared memory (denser frames: k6g)
  unsigned char* k6g;            // global-memory association layout for TCAP triples (K6Smem(SMAX, TCAP))
  // targets
  int32_t* det_target;           // [SMAX]  target index or -1
  int64_t* det_id;               // [SMAX]  instance id fused into (debug)
  uint32_t* tgt_phys;            // [SMAX]
  uint32_t* tgt_root;            // [SMAX]
  uint32_t* tgt_stage;           // [SMAX] new list entries appended this frame
  uint32_t* tgt_base;            // [SMAX] list length before the frame
  unsigned long long* tg_newoff; // [SMAX] arena offset of the (possibly moved) list
  unsigned long long* tg_movesrc;// [SMAX] old offset when K6 moved the list to a larger region, else ~0
  uint32_t* tg_mvoff;            // [SMAX+1] prefix offsets of the moved entries (K7 copy items)
  int32_t* ntgt;                 // [1]
  // per-target O12 work lists (written by K6, executed by K7a)
  int32_t* tg_kind;              // [SMAX] 0 = component with instances, 1 = new instance
  int64_t* tg_vbase;             // [SMAX] |V| of the physical owner
  uint32_t* tg_moff;             // [SMAX] offset into tg_mem (member ids ascending)
  uint32_t* tg_mcnt;
  uint32_t* tg_doff;             // [SMAX] offset into tg_dets (detections ascending)
  uint32_t* tg_dcnt;
  uint32_t* tg_mem;              // [TCAP]
  uint32_t* tg_dets;             // [SMAX]
  uint32_t* tg_cand;             // [SMAX][32] per target: members then detections (first 32), for K7's fast path
  // relabel segments
  uint32_t* seg_phys;            // [TCAP] old physical label
  int32_t* seg_tgt;              // [TCAP]
  uint32_t* seg_off;             // [TCAP+1] prefix offsets into the relabel item space
  unsigned long long* seg_base;  // [TCAP] arena offset of the old list
  int32_t* nseg;                 // [1]
  uint32_t* nrel;                // [1] total relabel items
  uint32_t* work;                // [1] K7 insert-chunk counter (zeroed by K6)
  disc_frame_report* rep;        // [MAXWIN] device reports
  int64_t* live_before;          // [1]
  // NEXT f2: per-frame active-set refinement (refine_active; k_refine).  RCAP = TCAP + SMAX active
  // instances at most, RPC-slot pair table
  unsigned long long* rf_pkey;   // [RPC] (i << 32 | j), i < j
  uint32_t* rf_pcnt;             // [RPC]
  int32_t RPC, RCAP;
  uint32_t* rf_act;              // [RCAP] active ids (unsorted), then ascending
  uint32_t* rf_act2;             // [RCAP]
  uint32_t* rf_n;                // [8]: 0 candidates, 1 edges, 2 components, 3 segments, 4 relabel items, 5 active
  uint32_t* rf_croot;            // [RCAP] component root id
  uint32_t* rf_cadd;             // [RCAP] new memberships of the root this round
  uint32_t* rf_cbase;            // [RCAP] root's list length before
  unsigned long long* rf_coff;   // [RCAP] root's list offset (after a move)
  uint32_t* rf_sL;               // [RCAP] relabel segment: member's physical label
  uint32_t* rf_sc;               // [RCAP]   its component
  unsigned long long* rf_sbase;  // [RCAP]   its key list offset
  uint32_t* rf_slen;             // [RCAP]   length
  uint32_t* rf_spre;             // [RCAP + 1] item prefix
  uint32_t* ntrip_last;          // [1] (debug export)
};

// per window slot: the frame's mask count and id (the sharded map's stage-2 kernels read them from
// device memory: a rank holds the inputs of its own frames only)
struct FrameMeta {
  int32_t S;
  int32_t pad;
  int64_t frame_id;
};

// ---- helpers -------------------------------------------------------------------------
// Fixed-point scales of a frame's pooling sums (powers of two: conversions are exact scalings before
// one rounding).  |w x| <= |r| xmax <= 2 sqrt(Df) xmax^2 per term (r = |f_p - fbar|), summed over <= P
// patches; the bound below (P 2 Df xmax^2) keeps every sum under 2^61.
__host__ __device__ __forceinline__ int pool_scale_exp(int P, int Df, float xmax, bool cover) {
  const double b = cover ? (double)P * (2.0 * (double)Df * (double)xmax + 1.0)
                         : (double)P * 2.0 * (double)Df * (double)xmax * (double)xmax;
  int e = 0;
  frexp(b + 1.0, &e);   // b + 1 < 2^e
  return 61 - e;
}
constexpr double ANG_SCALE = 1099511627776.0;   // 2^40: S_angle terms in [0, 1]
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
// owning shard of a voxel key in a G-way key-hash-sharded map: high hash bits, so
// ownership is independent of the slot position (low bits) inside the owner's hash table
__host__ __device__ __forceinline__ uint32_t key_owner(uint64_t key, uint32_t G) {
  return (uint32_t)((mix64(key) >> 40) % (uint64_t)G);
}
__device__ __forceinline__ uint64_t pack_key(int ix, int iy, int iz) {
  return ((uint64_t)(uint32_t)(ix + KEY_BIAS) << 42) | ((uint64_t)(uint32_t)(iy + KEY_BIAS) << 21) |
         (uint64_t)(uint32_t)(iz + KEY_BIAS);
}
__device__ __forceinline__ void unpack_key(uint64_t k, int& ix, int& iy, int& iz) {
  ix = (int)(k >> 42) - KEY_BIAS;
  iy = (int)((k >> 21) & 0x1FFFFF) - KEY_BIAS;
  iz = (int)(k & 0x1FFFFF) - KEY_BIAS;
}
__device__ __forceinline__ void raise_err(int* err, int code) { atomicMax(err, code); }
// -DDISC_BOUNDS: device-side bounds checks on the computed indices of the hot kernels (the check
// compute-sanitizer memcheck would do; that tool is closed on the GPU pool).  A violation prints
// the condition and raises DERR_BOUNDS, so the map's next synchronising call fails.
#ifdef DISC_BOUNDS
#define DBOUND(cond, err)                                                                    \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("DISC_BOUNDS %s:%d: %s\n", __FILE__, __LINE__, #cond);                          \
      raise_err((err), DERR_BOUNDS);                                                         \
    }                                                                                        \
  } while (0)
#else
#define DBOUND(cond, err) \
  do {                    \
  } while (0)
#endif
// internal invariant check: records 1000 + source line in the sticky error flag
#define DISC_CHECK(err, cond)                       \
  do {                                              \
    if (!(cond)) atomicCAS((err), 0, 1000 + __LINE__); \
  } while (0)

// dot_pin with every load of the lane issued before the (unchanged) fma chain
// R15 dot_pin, warp-cooperative (Dt <= 512): lane l accumulates d = l, l + 32, ... ascending with
// fma, then the xor butterfly 16, 8, 4, 2, 1 -- the oracle's ora_dot_pin order.
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

template <typename T>
__device__ __forceinline__ T vload(const T* p) {
  return *(const volatile T*)p;
}

}  // namespace disc
