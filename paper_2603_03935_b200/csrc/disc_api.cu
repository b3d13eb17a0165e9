// disc_api.cu -- libdisc's C ABI (include/disc.h): validation, device memory ownership,
// stream-ordered orchestration of the stage-1 window kernels and the per-frame stage-2
// kernels, error stickiness, exports.
//
// Every step of the hot path runs in the kernels of k_frame.cu / k_map.cu; this file only
// validates, sizes, launches and copies.
#include <cmath>
#include <dlfcn.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "disc_common.cuh"
#include "disc_launch.h"

using namespace disc;

struct EvPair {
  cudaEvent_t a, b;
  int kind;  // 0 = K1, 1 = stage 1, 2 = stage 2
};

struct disc_map {
  disc_config cfg;
  Params P;
  int dev = 0, nsm = 148;
  int nres = 0;       // SMs reserved for stage 2 (0 = no partition), windows with CLIP tokens
  int nres_geo = 0;   // the same for geometry-only windows (lighter stage 1: more SMs to stage 2)
  uint32_t s2_tag = 0;   // next slot-chain tag of stage 2's speculative counting (launch_stage2)
  int s2_spec = 2;       // stage 2's speculative work (DISC_S2_SPEC at creation): 2 counting, 1 slots, 0 hints
  MapState M{};
  WinBufs Wb[2]{};               // double-buffered window buffers (stage 1 of window w+1 overlaps
                                 // stage 2 of window w)
  int wbuf = 0, last_buf = 0;
  bool s2_pending[2] = {false, false};
  cudaStream_t s1 = nullptr, s2 = nullptr;   // internal streams: stage 1, stage 2
  cudaEvent_t ev_in = nullptr, ev_done = nullptr, ev_s1done = nullptr, ev_s1[2] = {nullptr, nullptr},
              ev_s2[2] = {nullptr, nullptr};
  FrameScratch X{};
  int* d_err = nullptr;
  int* h_err = nullptr;                 // pinned
  disc_frame_report* h_rep = nullptr;   // pinned [MAXWIN]
  // adaptive stage-2 reserve: each window's pair counts come back (pinned, no sync); a finished
  // copy sets the running pairs-per-frame level the next windows' SM split follows
  uint32_t* h_np = nullptr;             // pinned [2][MAXWIN]
  cudaEvent_t ev_np[2] = {nullptr, nullptr};
  int np_pending[2] = {0, 0};
  double np_avg = -1.0;
  bool adapt = true;
  std::vector<void*> allocs;
  disc_status sticky = DISC_OK;
  std::string err;
  cudaStream_t last_stream = nullptr;
  // last frame (debug export)
  bool have_last = false;
  int last_f = 0;
  FrameDesc last_fd{};
  bool last_sem = false;
  // timing
  bool timing = false;
  std::vector<EvPair> ev_pending;
  std::vector<cudaEvent_t> ev_pool;
  disc_stats stats{};
  // host-input staging: two window-sized buffers, so window w+1's H2D copies overlap window w's
  // kernels (ev_stage: stage 1 of the window that used the buffer is done reading it)
  uint8_t* stage = nullptr;           // the buffer being filled
  uint8_t* stage_buf[2] = {nullptr, nullptr};
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr};   // a staging buffer's H2D copies issued (on s0)
  cudaStream_t s0 = nullptr;                    // host-input copies: beside stage 1 and stage 2
  bool stage_pending[2] = {false, false};
  int stage_next = 0;
  size_t stage_bytes = 0;
  disc_frame_report* h_rep_all = nullptr;   // pinned, reports of a host-input call (copied once)
  int64_t h_rep_cap = 0;
  // export scratch
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // frame-table state per window buffer: clean = every slot EMPTY / zero (map creation; after a
  // window that released its slots); release when the tables are >= tab_ratio x the pairs per frame
  bool ktab_clean[2] = {true, true}, nsum_clean[2] = {true, true};
  double tab_ratio = 8.0;
  // key-hash-sharded map (world_size > 1): this handle drives the local shards (sub-maps)
  struct ShardGroup* grp = nullptr;
};

namespace {

const char* VERSION = "libdisc 0.1 (sm_100a)";

template <typename T>
T* dalloc(disc_map* m, size_t n, int fill = 0) {
  void* p = nullptr;
  const size_t b = n * sizeof(T) > 0 ? n * sizeof(T) : 16;
  if (cudaMalloc(&p, b) != cudaSuccess) return nullptr;
  cudaMemset(p, fill, b);
  m->allocs.push_back(p);
  return (T*)p;
}

uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

disc_status fail(disc_map* m, disc_status st, const std::string& msg) {
  if (m) {
    m->err = msg;
    if (st != DISC_ERR_INVALID) m->sticky = st;
  }
  return st;
}

disc_status cuda_check(disc_map* m, const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(m, DISC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return DISC_OK;
}

const char* dev_err_text(int code) {
  switch (code) {
    case DERR_FRAME_PAIRS: return "per-frame (mask, voxel) pair table full: raise max_pairs_per_frame";
    case DERR_MAP_KEYS: return "voxel hash full: raise max_memberships";
    case DERR_OVF_POOL: return "overflow label chunks exhausted: raise max_memberships";
    case DERR_ARENA: return "instance key-list arena exhausted: raise max_memberships";
    case DERR_TRIPLES: return "per-frame (segment, instance) count table full";
    case DERR_INSTANCES: return "max_instances exceeded";
    case DERR_STAGE: return "per-frame staging list full: raise max_memberships";
    case DERR_BOUNDS: return "internal index out of bounds (DISC_BOUNDS build)";
    default: {
      static thread_local char buf[96];
      if (code >= 1000) {
        std::snprintf(buf, sizeof(buf), "internal invariant violated (device check at source line %d)", code - 1000);
        return buf;
      }
      return "device error";
    }
  }
}

// synchronise the stream and surface device-side errors
disc_status sync_check(disc_map* m, cudaStream_t st) {
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(m, "cudaStreamSynchronize");
  if (cudaMemcpy(m->h_err, m->d_err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_check(m, "error flag");
  if (*m->h_err) return fail(m, *m->h_err >= 1000 ? DISC_ERR_INTERNAL : DISC_ERR_CAPACITY, dev_err_text(*m->h_err));
  return DISC_OK;
}

bool pose_rigid(const float* P) {   // A0, S:116-118 (same decision rule as documented in disc.h)
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(P[i])) return false;
  if (P[12] != 0.0f || P[13] != 0.0f || P[14] != 0.0f || P[15] != 1.0f) return false;
  double R[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = (double)P[4 * i + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double s = R[0][i] * R[0][j] + R[1][i] * R[1][j] + R[2][i] * R[2][j];
      if (std::fabs(s - (i == j ? 1.0 : 0.0)) > 1e-5) return false;
    }
  const double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                     R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                     R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  return std::fabs(det - 1.0) <= 1e-5;
}

std::string validate_frame(const disc_map* m, const disc_frame& f, bool host) {
  const disc_config& c = m->cfg;
  if (f.height <= 0 || f.width <= 0 || f.height > 65535 || f.width > 65535) return "bad image dims";
  if ((int64_t)f.height * f.width > c.max_pixels) return "H*W exceeds max_pixels";
  if (!f.depth) return "null depth";
  if (f.num_masks < 0 || f.num_masks > c.max_masks) return "num_masks outside [0, max_masks]";
  if (f.num_masks > 0 && !f.masks == !f.mask_bits) return "exactly one of masks / mask_bits must be given";
  if (f.patch_h < 1 || f.patch_h > f.height || f.patch_w < 1 || f.patch_w > f.width) return "bad patch grid";
  if ((int64_t)f.patch_h * f.patch_w > c.max_patches) return "Hp*Wp exceeds max_patches";
  if (f.patch_w > 65535) return "patch_w too large";
  if (c.track_dim > 0 && !f.track_feats) return "track_dim > 0 requires track_feats";
  if (!(f.fx != 0.0f && f.fy != 0.0f) || !std::isfinite(f.fx) || !std::isfinite(f.fy) || !std::isfinite(f.cx) ||
      !std::isfinite(f.cy))
    return "bad intrinsics";
  if (!pose_rigid(f.pose)) return "non-rigid pose";
  if (f.height > 16384 || f.width > 16384) return "frame dimension above 16384";
  (void)host;
  return "";
}

FrameDesc make_desc(const disc_frame& f) {
  FrameDesc d{};
  d.depth = f.depth;
  d.masks = f.masks;
  d.mbits = f.mask_bits;
  d.conf = f.mask_conf;
  d.feats = f.patch_feats;
  d.gemb = f.global_embed;
  d.track = f.track_feats;
  for (int i = 0; i < 12; ++i) d.pose[i] = f.pose[i];
  d.fx = f.fx; d.fy = f.fy; d.cx = f.cx; d.cy = f.cy;
  d.frame_id = f.frame_id;
  d.H = f.height; d.W = f.width; d.S = f.num_masks; d.Hp = f.patch_h; d.Wp = f.patch_w;
  // K1 reads mask planes with 32-byte loads and depth with 16-byte loads
  d.vec16 = (((int64_t)f.height * f.width) % 32 == 0) && (((uintptr_t)f.masks & 31) == 0) &&
            (((uintptr_t)f.depth & 15) == 0);
  return d;
}

cudaEvent_t ev_get(disc_map* m) {
  cudaEvent_t e;
  if (!m->ev_pool.empty()) {
    e = m->ev_pool.back();
    m->ev_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}

void collect_events(disc_map* m) {
  for (auto& p : m->ev_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    if (p.kind == 0) { m->stats.k1_ms += ms; m->stats.k1_launches++; }
    else if (p.kind == 1) m->stats.stage1_ms += ms;
    else m->stats.stage2_ms += ms;
    m->ev_pool.push_back(p.a);
    m->ev_pool.push_back(p.b);
  }
  m->ev_pending.clear();
}

}  // namespace

namespace disc {
// DISC_TIMELINE=1: an event after every launch (profiling aid; nsys is not in this image).
// tl_dump prints (stream, mark, frame, ms since the first mark) once the work has completed.
struct TlRec { cudaEvent_t ev; const char* name; int frame; cudaStream_t st; };
static std::vector<TlRec> g_tl;
static int tl_on() {
  static int on = -1;
  if (on < 0) on = getenv("DISC_TIMELINE") ? 1 : 0;
  return on;
}
void tl_mark(cudaStream_t st, const char* name, int frame) {
  if (!tl_on()) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_tl.push_back({e, name, frame, st});
}
void tl_dump() {
  if (!tl_on() || g_tl.empty()) return;
  cudaDeviceSynchronize();
  for (const TlRec& r : g_tl) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_tl[0].ev, r.ev);
    std::fprintf(stderr, "TL %p %s %d %.4f\n", (void*)r.st, r.name, r.frame, ms);
  }
  for (const TlRec& r : g_tl) cudaEventDestroy(r.ev);
  g_tl.clear();
}

void debug_check(cudaStream_t st, const char* kernel, int frame) {
  tl_mark(st, kernel, frame);
  static int on = -1;
  if (on < 0) on = getenv("DISC_DEBUG_SYNC") ? 1 : 0;
  if (!on) return;
  const cudaError_t e1 = cudaGetLastError();
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    std::fprintf(stderr, "DISC_DEBUG_SYNC: %s (frame %d): %s / %s\n", kernel, frame, cudaGetErrorString(e1),
                 cudaGetErrorString(e2));
}
}  // namespace disc

extern "C" {

const char* disc_version(void) { return VERSION; }

disc_status disc_nccl_unique_id(uint8_t out[128]) {
  if (!out) return DISC_ERR_INVALID;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) return DISC_ERR_NCCL;
  typedef int (*get_id_fn)(void*);   // ncclResult_t ncclGetUniqueId(ncclUniqueId*), 128-byte id
  get_id_fn get_id = (get_id_fn)dlsym(h, "ncclGetUniqueId");
  if (!get_id) return DISC_ERR_NCCL;
  unsigned char id[128];
  if (get_id(id) != 0) return DISC_ERR_NCCL;
  std::memcpy(out, id, 128);
  return DISC_OK;
}

disc_status disc_config_init(disc_config* c) {
  if (!c) return DISC_ERR_INVALID;
  std::memset(c, 0, sizeof(*c));
  c->voxel_size = 0.02f;
  c->tau_geo = 0.3f;
  c->tau_vis = 0.8f;
  c->depth_min = 0.1f;
  c->depth_max = 10.0f;
  c->mask_min_conf = 0.5f;
  c->mask_max_aspect = 10.0f;
  c->mask_min_area = 400;
  c->cover_min = 0.25f;
  c->lambda_size = 3.3f;
  c->eps_distinct = 1e-6f;
  c->dbscan_eps = 0.0f;      // R7: off unless asked for
  c->dbscan_min_pts = 8;
  c->refine_active = 0;      // R14 unless asked for (R43)
  c->feat_dim = 1024;
  c->track_dim = 384;
  c->max_memberships = 1ll << 22;
  c->max_instances = 1 << 16;
  c->max_masks = 64;
  c->max_pixels = 1280 * 720;
  c->max_patches = 8192;
  c->max_pairs_per_frame = 1 << 17;
  c->window = 16;
  c->device = 0;
  c->world_size = 1;
  c->rank = 0;
  c->nccl_unique_id = nullptr;
  return DISC_OK;
}

static std::string validate_config(const disc_config* c) {
  if (!(c->voxel_size > 0.0f) || !std::isfinite(c->voxel_size)) return "voxel_size must be > 0";
  if (!(c->tau_geo > 0.0f && c->tau_geo <= 1.0f)) return "tau_geo must be in (0,1]";
  if (!(c->tau_vis >= -1.0f && c->tau_vis <= 1.0f)) return "tau_vis must be in [-1,1]";
  if (!(c->depth_min >= 0.0f && c->depth_min < c->depth_max)) return "bad depth window";
  if (!(c->mask_min_conf >= 0.0f && c->mask_min_conf <= 1.0f)) return "mask_min_conf in [0,1]";
  if (!(c->mask_max_aspect >= 1.0f) || c->mask_min_area < 0) return "bad mask filter";
  if (!(c->cover_min >= 0.0f && c->cover_min <= 1.0f)) return "cover_min in [0,1]";
  if (!(c->lambda_size > 0.0f) || !(c->eps_distinct >= 0.0f)) return "bad lambda/eps";
  if (!(c->dbscan_eps >= 0.0f) || !std::isfinite(c->dbscan_eps) || (c->dbscan_eps > 0.0f && c->dbscan_min_pts < 1))
    return "dbscan_eps >= 0 (min_pts >= 1 when on)";
  if (c->feat_dim <= 0 || c->feat_dim % 4 != 0 || c->feat_dim > 1024)
    return "feat_dim must be a multiple of 4 in [4, 1024]";
  if (c->track_dim < 0 || c->track_dim > 512) return "track_dim must be in [0, 512]";
  if (c->max_masks < 1 || c->max_masks > 255) return "max_masks in [1,255]";
  if (c->max_pixels < 1 || c->max_patches < 1) return "bad max_pixels / max_patches";
  if (c->max_pairs_per_frame < 1 || c->max_pairs_per_frame > (1 << 22)) return "max_pairs_per_frame in [1, 2^22]";
  if (c->window < 1 || c->window > MAXWIN) return "window in [1,32]";
  if (c->refine_active != 0 && c->refine_active != 1) return "refine_active in {0, 1}";
  if (c->max_instances < 1 || c->max_instances > (1 << 30)) return "bad max_instances";
  // <= 2^28: the voxel hash (2^29 slots) and the key-list arena (8 * 2^28 + 2^20 entries) stay
  // indexable by 32-bit slot numbers / list offsets below the U32_EMPTY sentinel
  if (c->max_memberships < 1 || c->max_memberships > (1ll << 28)) return "max_memberships in [1, 2^28]";
  if (c->world_size != 1 || c->rank != 0) return "world_size / rank";   // (> 1: group_create)
  return "";
}

static disc_status group_create(const disc_config* cfg, disc_map** out);
static void group_destroy(disc_map* m);

disc_status disc_map_create(const disc_config* cfg, disc_map** out) {
  if (!cfg || !out) return DISC_ERR_INVALID;
  *out = nullptr;
  if (cfg->world_size > 1) return group_create(cfg, out);   // key-hash-sharded map
  const std::string v = validate_config(cfg);
  if (!v.empty()) {
    std::fprintf(stderr, "disc_map_create: %s\n", v.c_str());
    return DISC_ERR_INVALID;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
    cudaGetLastError();
    std::fprintf(stderr, "disc_map_create: no CUDA device %d\n", cfg->device);
    return DISC_ERR_CUDA;
  }
  cudaSetDevice(cfg->device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, cfg->device);
  if (prop.major != 10) {
    std::fprintf(stderr, "disc_map_create: libdisc is built for sm_100a (found sm_%d%d)\n", prop.major, prop.minor);
    return DISC_ERR_UNSUPPORTED;
  }
  disc_map* m = new disc_map();
  m->cfg = *cfg;
  m->dev = cfg->device;
  m->nsm = prop.multiProcessorCount;
  {  // stage-2 SM reserve; DISC_S2_SMS overrides it (tuning)
    const char* e = std::getenv("DISC_S2_SMS");
    // longer windows amortise stage 1's per-window work, so stage 2 gets a few more SMs (measured
    // on R: 16-frame windows best at 20, 32-frame windows at 26)
    m->nres = e ? std::atoi(e) : (cfg->window > 16 ? 26 : 20);
    m->nres = std::max(0, std::min(m->nres, m->nsm * 3 / 4));
    const char* eg = std::getenv("DISC_S2_SMS_GEO");
    m->nres_geo = eg ? std::atoi(eg) : (cfg->window > 16 ? 48 : 40);
    m->nres_geo = std::max(0, std::min(m->nres_geo, m->nsm * 3 / 4));
    const char* ea = std::getenv("DISC_S2_ADAPT");   // 0: fixed split (tuning)
    if (const char* es = std::getenv("DISC_S2_SPEC")) m->s2_spec = std::max(0, std::min(3, std::atoi(es)));
    m->adapt = !(ea && std::atoi(ea) == 0);
    const char* er = std::getenv("DISC_TAB_RELEASE_RATIO");   // tuning: 1e30 = always fill
    if (er) m->tab_ratio = std::atof(er);
  }
  Params& P = m->P;
  P.r = cfg->voxel_size; P.tau_geo = cfg->tau_geo; P.tau_vis = cfg->tau_vis;
  P.dmin = cfg->depth_min; P.dmax = cfg->depth_max; P.min_conf = cfg->mask_min_conf;
  P.max_aspect = cfg->mask_max_aspect; P.cover_min = cfg->cover_min; P.lambda = cfg->lambda_size;
  P.eps = cfg->eps_distinct; P.min_area = cfg->mask_min_area; P.Df = cfg->feat_dim; P.Dt = cfg->track_dim;
  P.db_eps = cfg->dbscan_eps; P.db_min = cfg->dbscan_min_pts; P.refine = cfg->refine_active;

  const int win = cfg->window, SM = cfg->max_masks, Df = cfg->feat_dim, Dt = cfg->track_dim;
  const int64_t PMAX = cfg->max_pairs_per_frame, PMP = cfg->max_patches;
  const int64_t PC = (int64_t)next_pow2(std::max<int64_t>(2 * PMAX, 1024));
  bool ok = true;
  auto chk = [&](void* p) { ok = ok && p; };
  // ---- window buffers ----
  for (int wbi = 0; wbi < 2; ++wbi) {
  WinBufs& W = m->Wb[wbi];
  W.PC = (int32_t)PC; W.PMAX = (int32_t)PMAX; W.SMAX = SM; W.PMAXP = (int32_t)PMP;
  W.RCAP = (int32_t)PMAX;
  if (const char* e = getenv("DISC_K1_RCAP")) W.RCAP = (int32_t)std::max<int64_t>(0, std::min<int64_t>(PMAX, atoll(e)));   // tests
  W.FCHUNKS = (int32_t)((PMP + 63) / 64);
  chk(W.ktab = dalloc<unsigned long long>(m, (size_t)win * PC, 0xFF));
  chk(W.ptab = dalloc<uint32_t>(m, (size_t)win * PC, 0xFF));
  chk(W.nsum = dalloc<NSum>(m, (size_t)win * PC, 0));
  chk(W.plist = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.npairs = dalloc<uint32_t>(m, win));
  chk(W.rkey = dalloc<unsigned long long>(m, (size_t)win * PMAX));
  chk(W.rs = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.rn = dalloc<NSum>(m, (size_t)win * PMAX));
  chk(W.rcount = dalloc<uint32_t>(m, win));
  chk(W.cnt = dalloc<uint32_t>(m, (size_t)win * SM * PMP));
  chk(W.area = dalloc<uint32_t>(m, (size_t)win * SM));
  chk(W.bbox = dalloc<int32_t>(m, (size_t)win * SM * 4));
  chk(W.vs = dalloc<uint32_t>(m, (size_t)win * SM));
  chk(W.daabb = dalloc<int32_t>(m, (size_t)win * SM * 6));
  chk(W.ang64 = dalloc<unsigned long long>(m, (size_t)win * SM));
  chk(W.pw = dalloc<uint32_t>(m, (size_t)win * SM));
  chk(W.xmax = dalloc<float>(m, (size_t)win));
  chk(W.ang_cnt = dalloc<uint32_t>(m, (size_t)win * SM));
  chk(W.oor = dalloc<unsigned long long>(m, win));
  chk(W.pkey = dalloc<unsigned long long>(m, (size_t)win * PMAX));
  chk(W.pinfo = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.pfk = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.pms = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.plab = dalloc<uint2>(m, (size_t)win * PMAX));
  chk(W.pnext = dalloc<uint32_t>(m, (size_t)win * PMAX));
  chk(W.fpart = dalloc<double>(m, (size_t)win * W.FCHUNKS * Df));
  chk(W.fbar = dalloc<float>(m, (size_t)win * Df));
  chk(W.rp = dalloc<float>(m, (size_t)win * PMP));
  chk(W.rbar = dalloc<double>(m, (size_t)win));
  chk(W.psum64 = dalloc<long long>(m, (size_t)win * SM * 3));
  chk(W.status = dalloc<int32_t>(m, (size_t)win * SM));
  chk(W.qf = dalloc<float>(m, (size_t)win * SM * 6));
  chk(W.emb = dalloc<float>(m, (size_t)win * SM * Df));
  chk(W.emb64 = dalloc<long long>(m, (size_t)win * SM * Df));
  chk(W.trk = dalloc<double>(m, (size_t)win * SM * std::max(Dt, 1)));
  chk(W.tok = dalloc<uint8_t>(m, (size_t)win * SM));
  chk(W.pmode = dalloc<uint8_t>(m, (size_t)win * SM));
  chk(W.k1ctr = dalloc<uint32_t>(m, 2));
  if (cfg->dbscan_eps > 0.0f) {   // NEXT f3: per-frame (mask, point) records of the DBSCAN denoise
    // (overlapping masks put a pixel into several masks' clouds: up to 8 per pixel, or PMAX)
    W.DBP = (int32_t)std::min<int64_t>(1 << 24, std::max<int64_t>((int64_t)std::min(SM, 8) * cfg->max_pixels, PMAX));
    const size_t nd = (size_t)win * W.DBP;
    chk(W.dbk = dalloc<unsigned long long>(m, nd));
    chk(W.dbv = dalloc<uint32_t>(m, nd));
    chk(W.dbk2 = dalloc<unsigned long long>(m, nd));
    chk(W.dbv2 = dalloc<uint32_t>(m, nd));
    chk(W.dbx = dalloc<float4>(m, nd));
    chk(W.dbpar = dalloc<uint32_t>(m, nd));
    chk(W.dblab = dalloc<uint32_t>(m, nd));
    chk(W.dbsz = dalloc<uint32_t>(m, nd));
    chk(W.dbcore = dalloc<uint8_t>(m, nd));
    chk(W.dbbest = dalloc<unsigned long long>(m, (size_t)win * SM));
    chk(W.dbn = dalloc<uint32_t>(m, win));
    chk(W.dbbeg = dalloc<int>(m, win));
    chk(W.dbend = dalloc<int>(m, win));
    W.dbtmp_bytes = dbscan_tmp_bytes((int)nd, win);
    chk(W.dbtmp = dalloc<unsigned char>(m, W.dbtmp_bytes));
  }
  W.MPIX = ((int64_t)cfg->max_pixels + 31) / 32 * 32;   // flat per-frame maps, sector-aligned
  chk(W.m0map = dalloc<uint16_t>(m, (size_t)win * W.MPIX));
  chk(W.s2bar = dalloc<uint32_t>(m, 1));
  }
  {  // K1 normal-sum scratch, shared by both window buffers (K1 launches are stream-ordered)
    const int nsmid = k1_nsmid();
    NSum* scr = dalloc<NSum>(m, (size_t)nsmid * K1_SLOTS_PER_SM * K1_PT, 0);
    uint32_t* slot = dalloc<uint32_t>(m, (size_t)nsmid, 0);
    chk(scr); chk(slot);
    uint32_t* s2sm = dalloc<uint32_t>(m, 8, 0);
    chk(s2sm);
    for (int wbi = 0; wbi < 2; ++wbi) { m->Wb[wbi].k1scr = scr; m->Wb[wbi].k1slot = slot; m->Wb[wbi].s2sm = s2sm; }
  }
  // ---- map ----
  MapState& M = m->M;
  const int64_t IM = cfg->max_instances;
  M.MC = next_pow2(std::max<int64_t>(2 * cfg->max_memberships, 1024));
  M.OVFCAP = (uint32_t)std::max<int64_t>(4096, cfg->max_memberships / 8);
  M.ARENA = (unsigned long long)(8 * cfg->max_memberships + (1 << 20));
  M.IMAX = (int32_t)IM;
  chk(M.slots = dalloc<KeySlot>(m, M.MC, 0xFF));
  chk(M.slh = dalloc<unsigned long long>(m, M.MC, 0));
  chk(M.ovf = dalloc<OvfChunk>(m, M.OVFCAP, 0xFF));
  chk(M.ovf_top = dalloc<uint32_t>(m, 1));
  chk(M.alive = dalloc<uint8_t>(m, IM));
  chk(M.phys_of = dalloc<uint32_t>(m, IM, 0xFF));
  chk(M.id_of = dalloc<uint32_t>(m, IM, 0xFF));
  chk(M.vcount = dalloc<int64_t>(m, IM));
  chk(M.obs = dalloc<int32_t>(m, IM));
  chk(M.last_seen = dalloc<int64_t>(m, IM));
  chk(M.aabb = dalloc<int32_t>(m, IM * 6));
  chk(M.q = dalloc<float>(m, IM));
  chk(M.E = dalloc<float>(m, (size_t)IM * Df));
  chk(M.T = dalloc<double>(m, (size_t)IM * std::max(Dt, 1)));
  chk(M.TT = dalloc<double>(m, IM));
  chk(M.lst_off = dalloc<unsigned long long>(m, IM));
  chk(M.lst_len = dalloc<uint32_t>(m, IM));
  chk(M.lst_cap = dalloc<uint32_t>(m, IM));
  chk(M.arena = dalloc<uint32_t>(m, M.ARENA));
  chk(M.arena_top = dalloc<unsigned long long>(m, 1));
  chk(M.stamp = dalloc<uint32_t>(m, IM));
  chk(M.local = dalloc<int32_t>(m, IM));
  chk(M.counters = dalloc<int64_t>(m, 8));
  chk(m->d_err = dalloc<int>(m, 1));
  M.err = m->d_err;
  // ---- per-frame scratch ----
  FrameScratch& X = m->X;
  // (s, j) count triples per frame: up to TCS in the association's shared-memory tables, up to
  // TCAP through its global-memory layout (dense SAM-"everything" frames: ~S^2/10 triples measured
  // at S = 150); DISC_TCAP / DISC_K6_TCS override them (tests force the global layout with TCS 0)
  X.TCS = 3072;
  X.TCAP = (int32_t)std::max<int64_t>(X.TCS, (int64_t)SM * 256);
  if (const char* e = getenv("DISC_TCAP")) X.TCAP = std::max(1, atoi(e));
  if (const char* e = getenv("DISC_K6_TCS")) X.TCS = std::max(0, std::min(3072, atoi(e)));
  X.CC = (int32_t)next_pow2(std::max<int64_t>(16384, 2 * (int64_t)X.TCAP));
  chk(X.k6g = dalloc<unsigned char>(m, k6_layout_bytes(SM, X.TCAP)));
  chk(X.ctab_key = dalloc<unsigned long long>(m, X.CC, 0xFF));
  chk(X.ctab_cnt = dalloc<uint32_t>(m, X.CC));
  chk(X.ctab_idx = dalloc<uint32_t>(m, X.TCAP));
  chk(X.ntrip = dalloc<uint32_t>(m, 1));
  chk(X.trip_gate = dalloc<uint8_t>(m, X.TCAP));
  chk(X.gate_done = dalloc<uint32_t>(m, 1, 0));
  chk(X.trip_s = dalloc<uint32_t>(m, X.TCAP));
  chk(X.trip_j = dalloc<uint32_t>(m, X.TCAP));
  chk(X.trip_c = dalloc<uint32_t>(m, X.TCAP));
  chk(X.trip_edge = dalloc<uint8_t>(m, X.TCAP));
  chk(X.trip_sd = dalloc<uint32_t>(m, X.TCAP));
  chk(X.trip_jd = dalloc<uint32_t>(m, X.TCAP));
  chk(X.ctab_key2 = dalloc<unsigned long long>(m, X.CC, 0xFF));
  chk(X.ctab_cnt2 = dalloc<uint32_t>(m, X.CC));
  chk(X.ctab_idx2 = dalloc<uint32_t>(m, X.TCAP));
  chk(X.ntrip2 = dalloc<uint32_t>(m, 1));
  chk(X.trip_s2 = dalloc<uint32_t>(m, X.TCAP));
  chk(X.trip_j2 = dalloc<uint32_t>(m, X.TCAP));
  chk(X.det_target = dalloc<int32_t>(m, SM));
  chk(X.det_id = dalloc<int64_t>(m, SM));
  chk(X.tgt_phys = dalloc<uint32_t>(m, SM));
  chk(X.tgt_root = dalloc<uint32_t>(m, SM));
  chk(X.tgt_stage = dalloc<uint32_t>(m, SM));
  chk(X.tg_newoff = dalloc<unsigned long long>(m, SM));
  chk(X.tg_movesrc = dalloc<unsigned long long>(m, SM));
  chk(X.tg_mvoff = dalloc<uint32_t>(m, SM + 1));
  chk(X.tgt_base = dalloc<uint32_t>(m, SM));
  chk(X.ntgt = dalloc<int32_t>(m, 1));
  chk(X.tg_kind = dalloc<int32_t>(m, SM));
  chk(X.tg_vbase = dalloc<int64_t>(m, SM));
  chk(X.tg_moff = dalloc<uint32_t>(m, SM));
  chk(X.tg_mcnt = dalloc<uint32_t>(m, SM));
  chk(X.tg_doff = dalloc<uint32_t>(m, SM));
  chk(X.tg_dcnt = dalloc<uint32_t>(m, SM));
  chk(X.tg_mem = dalloc<uint32_t>(m, X.TCAP));
  chk(X.tg_dets = dalloc<uint32_t>(m, SM));
  chk(X.tg_cand = dalloc<uint32_t>(m, (size_t)SM * 32));
  chk(X.seg_phys = dalloc<uint32_t>(m, X.TCAP));
  chk(X.seg_tgt = dalloc<int32_t>(m, X.TCAP));
  chk(X.seg_off = dalloc<uint32_t>(m, X.TCAP + 1));
  chk(X.seg_base = dalloc<unsigned long long>(m, X.TCAP));
  chk(X.nseg = dalloc<int32_t>(m, 1));
  chk(X.nrel = dalloc<uint32_t>(m, 1));
  chk(X.work = dalloc<uint32_t>(m, 1));
  chk(X.rep = dalloc<disc_frame_report>(m, MAXWIN));
  if (cfg->refine_active) {   // NEXT f2 buffers (k_refine)
    X.RCAP = X.TCAP + SM;
    X.RPC = (int32_t)next_pow2(std::max<int64_t>(1 << 16, 4 * (int64_t)X.RCAP));
    chk(X.rf_pkey = dalloc<unsigned long long>(m, X.RPC, 0xFF));
    chk(X.rf_pcnt = dalloc<uint32_t>(m, X.RPC));
    chk(X.rf_act = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_act2 = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_n = dalloc<uint32_t>(m, 8));
    chk(X.rf_croot = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_cadd = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_cbase = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_coff = dalloc<unsigned long long>(m, X.RCAP));
    chk(X.rf_sL = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_sc = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_sbase = dalloc<unsigned long long>(m, X.RCAP));
    chk(X.rf_slen = dalloc<uint32_t>(m, X.RCAP));
    chk(X.rf_spre = dalloc<uint32_t>(m, X.RCAP + 1));
  }
  chk(X.live_before = dalloc<int64_t>(m, 1));
  chk(X.ntrip_last = dalloc<uint32_t>(m, 1));
  {
    int prio_lo = 0, prio_hi = 0;   // stage 2 (latency-bound, few SMs) gets the higher priority
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&m->s1, cudaStreamNonBlocking, prio_lo) != cudaSuccess) ok = false;
    if (cudaStreamCreateWithPriority(&m->s2, cudaStreamNonBlocking, prio_hi) != cudaSuccess) ok = false;
  }
  for (cudaEvent_t* e : {&m->ev_in, &m->ev_done, &m->ev_s1done, &m->ev_s1[0], &m->ev_s1[1], &m->ev_s2[0], &m->ev_s2[1],
                         &m->ev_np[0], &m->ev_np[1]})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) ok = false;
  if (cudaMallocHost(&m->h_np, sizeof(uint32_t) * 2 * MAXWIN) != cudaSuccess) ok = false;
  if (cudaMallocHost(&m->h_err, sizeof(int)) != cudaSuccess) ok = false;
  if (cudaMallocHost(&m->h_rep, sizeof(disc_frame_report) * MAXWIN) != cudaSuccess) ok = false;
  if (ok && k6_smem_bytes(SM, X.TCS) > 227 * 1024) ok = false;
  cudaDeviceSynchronize();
  if (!ok || cudaGetLastError() != cudaSuccess) {
    std::fprintf(stderr, "disc_map_create: device allocation failed\n");
    disc_map_destroy(m);
    return DISC_ERR_CAPACITY;
  }
  *m->h_err = 0;
  *out = m;
  return DISC_OK;
}

void disc_map_destroy(disc_map* m) {
  if (!m) return;
  cudaSetDevice(m->dev);
  cudaDeviceSynchronize();
  group_destroy(m);
  for (void* p : m->allocs) cudaFree(p);
  if (m->h_err) cudaFreeHost(m->h_err);
  if (m->h_rep) cudaFreeHost(m->h_rep);
  if (m->h_np) cudaFreeHost(m->h_np);
  for (int i = 0; i < 2; ++i) {
    if (m->stage_buf[i]) cudaFree(m->stage_buf[i]);
    if (m->ev_stage[i]) cudaEventDestroy(m->ev_stage[i]);
    if (m->ev_h2d[i]) cudaEventDestroy(m->ev_h2d[i]);
  }
  if (m->s0) cudaStreamDestroy(m->s0);
  if (m->h_rep_all) cudaFreeHost(m->h_rep_all);
  if (m->scratch) cudaFree(m->scratch);
  for (auto& p : m->ev_pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : m->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : {m->ev_in, m->ev_done, m->ev_s1done, m->ev_s1[0], m->ev_s1[1], m->ev_s2[0], m->ev_s2[1],
                        m->ev_np[0], m->ev_np[1]})
    if (e) cudaEventDestroy(e);
  if (m->s1) cudaStreamDestroy(m->s1);
  if (m->s2) cudaStreamDestroy(m->s2);
  delete m;
}

// ==========================================================================================
// Key-hash-sharded map.  G shards; shard g owns the voxel keys with
// key_owner(key, G) == g (their memberships, hash slots and per-instance key lists) and a replica
// of the instance table.  Per window: stage 1 frame-parallel (shard g runs window slots g + G j),
// the detection records all-gathered, every kept (s, key) pair routed to its owner; per frame:
// lookup on own keys -> X1 all-gather of the partial (s, label, count) triples, each shard adds
// the others' into its count table (integer sums: identical on every shard) -> the association,
// replicated (identical decisions) -> apply on own keys, instance updates on every replica ->
// X2 all-reduce of the new memberships per target -> |V| and the report.
//  * one process, G shards on one device (nccl_unique_id == NULL): the exchanges are device copies;
//  * G processes (torchrun, one GPU each), one shard per rank: the exchanges are NCCL collectives
//    (ncclAllGather / ncclAllReduce / grouped ncclSend + ncclRecv) on the caller's stream.
// ==========================================================================================
static disc_status ensure_stage(disc_map* m);
static void stage_frame(disc_map* m, size_t& so, disc_frame& f, cudaStream_t st);

struct NcclApi {
  struct UniqueId { char internal[128]; };
  void* lib = nullptr;
  int (*init_rank)(void**, int, UniqueId, int) = nullptr;
  int (*destroy)(void*) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*errstr)(int) = nullptr;
  enum { U8 = 1, U32 = 3, I64 = 4, U64 = 5, SUM = 0 };
  bool load() {
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) return false;
    init_rank = (decltype(init_rank))dlsym(lib, "ncclCommInitRank");
    destroy = (decltype(destroy))dlsym(lib, "ncclCommDestroy");
    all_gather = (decltype(all_gather))dlsym(lib, "ncclAllGather");
    all_reduce = (decltype(all_reduce))dlsym(lib, "ncclAllReduce");
    send = (decltype(send))dlsym(lib, "ncclSend");
    recv = (decltype(recv))dlsym(lib, "ncclRecv");
    group_start = (decltype(group_start))dlsym(lib, "ncclGroupStart");
    group_end = (decltype(group_end))dlsym(lib, "ncclGroupEnd");
    errstr = (decltype(errstr))dlsym(lib, "ncclGetErrorString");
    return init_rank && destroy && all_gather && all_reduce && send && recv && group_start && group_end;
  }
};

struct ShardGroup {
  int G = 1;          // shards in total
  int L = 1;          // shards in this process (one process: G; NCCL: 1)
  int rank = 0;       // NCCL rank (this process's shard = rank); 0 in one process
  bool nccl = false;
  std::vector<disc_map*> sh;   // local shards (complete single maps: state, window buffers, scratch)
  DetLayout DL{1, 4, 0};
  int nloc = 1;                // frames per shard per window
  uint8_t* det_send = nullptr; // [nloc][REC] (NCCL)
  uint8_t* det_all = nullptr;  // [G][nloc][REC]
  uint32_t* trip_all = nullptr;
  size_t trip_stride = 0;      // u32 per shard: 1 + 3 TCAP
  int64_t* add_all = nullptr;  // [G][SMAX + 2]
  size_t add_stride = 0;
  FrameMeta* meta = nullptr;   // [window] (device)
  FrameMeta* h_meta = nullptr; // pinned [window]
  RouteDst* route = nullptr;   // device: local shards' stage-2 pair arrays
  // NCCL pair all-to-all
  NcclApi nc;
  void* comm = nullptr;
  PairRec* psend = nullptr;
  PairRec* precv = nullptr;
  size_t pcap = 0;
  unsigned long long* pcnt = nullptr;   // [G] counts, then scatter cursors
  unsigned long long* poff = nullptr;   // [G] send offsets
  unsigned long long* pmat = nullptr;   // [G][G] count matrix (all-gathered)
  unsigned long long* h_pmat = nullptr; // pinned [G][G]
  disc_frame_report* h_rep = nullptr;   // pinned [window]
};

static disc_status group_fail_nccl(disc_map* m, int rc, const char* what) {
  ShardGroup& Gp = *m->grp;
  return fail(m, DISC_ERR_NCCL, std::string(what) + ": " + (Gp.nc.errstr ? Gp.nc.errstr(rc) : "nccl error"));
}

static void group_destroy(disc_map* m) {
  ShardGroup* g = m->grp;
  if (!g) return;
  for (disc_map* s : g->sh) disc_map_destroy(s);
  if (g->comm && g->nc.destroy) g->nc.destroy(g->comm);
  if (g->h_meta) cudaFreeHost(g->h_meta);
  if (g->h_pmat) cudaFreeHost(g->h_pmat);
  if (g->h_rep) cudaFreeHost(g->h_rep);
  delete g;
  m->grp = nullptr;
}

static disc_status group_create(const disc_config* cfg, disc_map** out) {
  const int G = cfg->world_size;
  if (cfg->refine_active) return DISC_ERR_UNSUPPORTED;   // (the refinement's key lists span every shard)
  const bool nccl = cfg->nccl_unique_id != nullptr;
  if (G < 2 || G > MAX_LOCAL_SHARDS * 64) return DISC_ERR_INVALID;
  if (nccl ? (cfg->rank < 0 || cfg->rank >= G) : (cfg->rank != 0 || G > MAX_LOCAL_SHARDS)) return DISC_ERR_INVALID;
  disc_config sc = *cfg;
  sc.world_size = 1;
  sc.rank = 0;
  sc.nccl_unique_id = nullptr;
  const std::string v = validate_config(&sc);
  if (!v.empty()) {
    std::fprintf(stderr, "disc_map_create: %s\n", v.c_str());
    return DISC_ERR_INVALID;
  }
  disc_map* m = new disc_map();
  m->cfg = *cfg;
  m->dev = cfg->device;
  m->grp = new ShardGroup();
  ShardGroup& Gp = *m->grp;
  Gp.G = G;
  Gp.nccl = nccl;
  Gp.L = nccl ? 1 : G;
  Gp.rank = nccl ? cfg->rank : 0;
  for (int l = 0; l < Gp.L; ++l) {
    disc_map* s = nullptr;
    const disc_status st = disc_map_create(&sc, &s);
    if (st != DISC_OK) {
      disc_map_destroy(m);
      return st;
    }
    Gp.sh.push_back(s);
  }
  cudaSetDevice(cfg->device);
  m->nsm = Gp.sh[0]->nsm;
  const int SM = cfg->max_masks, Df = cfg->feat_dim, Dt = cfg->track_dim, win = cfg->window;
  Gp.DL = DetLayout(SM, Df, Dt);
  Gp.nloc = nccl ? std::max(1, win / G) : (win + G - 1) / G;
  const size_t rec = Gp.DL.total;
  bool ok = true;
  auto chk = [&](void* p) { ok = ok && p; };
  chk(Gp.det_all = dalloc<uint8_t>(m, (size_t)G * Gp.nloc * rec));
  if (nccl) chk(Gp.det_send = dalloc<uint8_t>(m, (size_t)Gp.nloc * rec));
  const int TCAP = Gp.sh[0]->X.TCAP;
  Gp.trip_stride = 1 + 3 * (size_t)TCAP;
  chk(Gp.trip_all = dalloc<uint32_t>(m, (size_t)G * Gp.trip_stride));
  Gp.add_stride = (size_t)SM + 2;
  chk(Gp.add_all = dalloc<int64_t>(m, (size_t)G * Gp.add_stride));
  chk(Gp.meta = dalloc<FrameMeta>(m, (size_t)MAXWIN));
  chk(Gp.route = dalloc<RouteDst>(m, 1));
  if (cudaMallocHost(&Gp.h_meta, sizeof(FrameMeta) * MAXWIN) != cudaSuccess) ok = false;
  if (cudaMallocHost(&Gp.h_rep, sizeof(disc_frame_report) * MAXWIN) != cudaSuccess) ok = false;
  if (ok) {
    RouteDst rd{};
    for (int l = 0; l < Gp.L; ++l) {
      const WinBufs& w = Gp.sh[l]->Wb[1];
      rd.pkey[l] = w.pkey;
      rd.pinfo[l] = w.pinfo;
      rd.npairs[l] = w.npairs;
    }
    rd.PMAX = Gp.sh[0]->Wb[1].PMAX;
    cudaMemcpy(Gp.route, &rd, sizeof(rd), cudaMemcpyHostToDevice);
  }
  if (ok && nccl) {
    // pair all-to-all buffers: a rank's frames of one window hold at most nloc * PMAX pairs
    Gp.pcap = (size_t)Gp.nloc * cfg->max_pairs_per_frame;
    chk(Gp.psend = dalloc<PairRec>(m, Gp.pcap));
    chk(Gp.precv = dalloc<PairRec>(m, Gp.pcap * G));
    chk(Gp.pcnt = dalloc<unsigned long long>(m, G));
    chk(Gp.poff = dalloc<unsigned long long>(m, G));
    chk(Gp.pmat = dalloc<unsigned long long>(m, (size_t)G * G));
    if (cudaMallocHost(&Gp.h_pmat, sizeof(unsigned long long) * G * G) != cudaSuccess) ok = false;
    if (ok && !Gp.nc.load()) {
      std::fprintf(stderr, "disc_map_create: libnccl.so.2 not loadable\n");
      disc_map_destroy(m);
      return DISC_ERR_NCCL;
    }
    if (ok) {
      NcclApi::UniqueId id;
      std::memcpy(id.internal, cfg->nccl_unique_id, 128);
      const int rc = Gp.nc.init_rank(&Gp.comm, G, id, cfg->rank);
      if (rc != 0) {
        std::fprintf(stderr, "disc_map_create: ncclCommInitRank failed (%d)\n", rc);
        disc_map_destroy(m);
        return DISC_ERR_NCCL;
      }
    }
  }
  if (cudaEventCreateWithFlags(&m->ev_done, cudaEventDisableTiming) != cudaSuccess) ok = false;
  cudaDeviceSynchronize();
  if (!ok || cudaGetLastError() != cudaSuccess) {
    std::fprintf(stderr, "disc_map_create: device allocation failed (sharded map)\n");
    disc_map_destroy(m);
    return DISC_ERR_CAPACITY;
  }
  *out = m;
  return DISC_OK;
}

// surface device errors of every local shard (sticky)
static disc_status group_sync(disc_map* m, cudaStream_t st) {
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(m, "cudaStreamSynchronize");
  for (disc_map* s : m->grp->sh) {
    const disc_status r = sync_check(s, st);
    if (r != DISC_OK) return fail(m, r, s->err);
  }
  return DISC_OK;
}

// n = frames of THIS caller (one process: the whole stream, window slot i = frame w0 + i, shard
// g runs the slots i = g mod G; NCCL: this rank's frames, global slot rank + G j = its frame w0 + j)
static disc_status group_integrate(disc_map* m, const disc_frame* frames, int32_t n, void* stream,
                                   disc_frame_report* reports, bool host_inputs) {
  if (!m || (!frames && n > 0) || n < 0) return DISC_ERR_INVALID;
  if (m->sticky != DISC_OK) return m->sticky;
  ShardGroup& Gp = *m->grp;
  cudaSetDevice(m->dev);
  cudaStream_t st = (cudaStream_t)stream;
  m->last_stream = st;
  for (int i = 0; i < n; ++i) {   // O0 over every frame before any mutation
    const std::string v = validate_frame(m, frames[i], host_inputs);
    if (!v.empty()) return fail(m, DISC_ERR_INVALID, "frame " + std::to_string(i) + ": " + v);
  }
  const int G = Gp.G, L = Gp.L, SM = m->cfg.max_masks, Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  const int per_call = Gp.nccl ? Gp.nloc : m->cfg.window;   // caller frames per window
  for (int w0 = 0; w0 < n; w0 += per_call) {
    const int nc = std::min(per_call, n - w0);
    const int Wn = Gp.nccl ? G * nc : nc;   // window slots
    // stage 1 and the record packing follow this process's own frames; the replicated stage 2
    // (and the unpacking) must assume tokens when another rank's frames may carry them (NCCL): a
    // frame without tokens has q = -1 everywhere, so no embedding is ever taken from it
    bool sem_own = false;
    for (int i = 0; i < nc; ++i) sem_own = sem_own || frames[w0 + i].patch_feats != nullptr;
    const bool sem = Gp.nccl || sem_own;
    // ---- stage 1, frame-parallel: local shard l (global g) runs its window slots ----
    for (int l = 0; l < L; ++l) {
      disc_map* s = Gp.sh[l];
      const int g = Gp.nccl ? Gp.rank : l;
      if (host_inputs) {
        const disc_status ss = ensure_stage(s);
        if (ss != DISC_OK) return fail(m, ss, s->err);
      }
      WinDesc wd{};
      wd.Df = Df;
      wd.Dt = Dt;
      int maxS = 1, maxP = 1;
      size_t so = 0;
      for (int j = 0;; ++j) {
        const int ci = Gp.nccl ? j : g + G * j;   // caller frame index within the window
        if (ci >= nc) break;
        disc_frame f = frames[w0 + ci];
        if (host_inputs) stage_frame(s, so, f, st);
        wd.f[wd.n] = make_desc(f);
        Gp.h_meta[wd.n] = FrameMeta{f.num_masks, 0, f.frame_id};
        maxS = std::max(maxS, f.num_masks);
        maxP = std::max(maxP, f.patch_h * f.patch_w);
        m->stats.mask_bytes += (int64_t)f.height * f.width * f.num_masks;
        m->stats.depth_bytes += (int64_t)f.height * f.width * 4;
        m->stats.track_bytes += (int64_t)f.patch_h * f.patch_w * Dt * 2;
        if (f.patch_feats) m->stats.feat_bytes += (int64_t)f.patch_h * f.patch_w * Df * 4;
        wd.n++;
      }
      cudaMemsetAsync(s->Wb[1].npairs, 0, sizeof(uint32_t) * m->cfg.window, st);
      if (wd.n > 0) {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (m->timing && l == 0) { e0 = ev_get(m); e1 = ev_get(m); }
        m->stats.launches += launch_stage1(wd, s->Wb[0], s->P, s->d_err, sem_own, maxS, 1, 1, 1, maxP, 4, s->nsm, 0,
                                           st, e0, e1);
        if (e0) m->ev_pending.push_back({e0, e1, 0});
        uint8_t* dst = Gp.nccl ? Gp.det_send : Gp.det_all + (size_t)g * Gp.nloc * Gp.DL.total;
        launch_det_pack(s->Wb[0], wd.n, Gp.h_meta, dst, Gp.DL, Df, Dt, sem_own, st);
      }
      // (the pinned meta is read at launch: kernel arguments are copied by value)
    }
    // ---- stage-1 exchange: detection records to every shard, pairs to their owners ----
    if (Gp.nccl) {
      int rc = Gp.nc.all_gather(Gp.det_send, Gp.det_all, (size_t)Gp.nloc * Gp.DL.total, NcclApi::U8, Gp.comm, st);
      if (rc) return group_fail_nccl(m, rc, "ncclAllGather(detections)");
      disc_map* s = Gp.sh[0];
      cudaMemsetAsync(Gp.pcnt, 0, sizeof(unsigned long long) * G, st);
      launch_pair_route(s->Wb[0], nc, Gp.rank, G, nullptr, Gp.pcnt, nullptr, nullptr, s->d_err, st);
      rc = Gp.nc.all_gather(Gp.pcnt, Gp.pmat, G, NcclApi::U64, Gp.comm, st);
      if (rc) return group_fail_nccl(m, rc, "ncclAllGather(pair counts)");
      cudaMemcpyAsync(Gp.h_pmat, Gp.pmat, sizeof(unsigned long long) * G * G, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);   // the all-to-all sizes (one host round trip per window)
      std::vector<unsigned long long> off(G), roff(G + 1, 0);
      unsigned long long o = 0;
      for (int d = 0; d < G; ++d) { off[d] = o; o += Gp.h_pmat[(size_t)Gp.rank * G + d]; }
      for (int r = 0; r < G; ++r) roff[r + 1] = roff[r] + Gp.h_pmat[(size_t)r * G + Gp.rank];
      if (o > Gp.pcap || roff[G] > Gp.pcap * G) return fail(m, DISC_ERR_CAPACITY, "pair exchange buffer full");
      cudaMemcpyAsync(Gp.poff, off.data(), sizeof(unsigned long long) * G, cudaMemcpyHostToDevice, st);
      cudaMemsetAsync(Gp.pcnt, 0, sizeof(unsigned long long) * G, st);
      launch_pair_route(s->Wb[0], nc, Gp.rank, G, nullptr, Gp.pcnt, Gp.poff, Gp.psend, s->d_err, st);
      Gp.nc.group_start();
      for (int r = 0; r < G; ++r) {
        const unsigned long long ns = Gp.h_pmat[(size_t)Gp.rank * G + r], nr = Gp.h_pmat[(size_t)r * G + Gp.rank];
        if (ns) Gp.nc.send(Gp.psend + off[r], ns * sizeof(PairRec), NcclApi::U8, r, Gp.comm, st);
        if (nr) Gp.nc.recv(Gp.precv + roff[r], nr * sizeof(PairRec), NcclApi::U8, r, Gp.comm, st);
      }
      rc = Gp.nc.group_end();
      if (rc) return group_fail_nccl(m, rc, "ncclSend/ncclRecv(pairs)");
      launch_pair_deliver(Gp.precv, roff[G], s->Wb[1], s->d_err, st);
    } else {
      for (int l = 0; l < L; ++l) {
        const int nown = (nc - l + G - 1) / G;
        launch_pair_route(Gp.sh[l]->Wb[0], nown, l, G, Gp.route, nullptr, nullptr, nullptr, Gp.sh[l]->d_err, st);
      }
    }
    for (int l = 0; l < L; ++l)
      launch_det_unpack(Gp.det_all, Wn, G, Gp.nloc, Gp.DL, Gp.sh[l]->Wb[1], Gp.meta, Df, Dt, sem, st);
    // ---- stage 2, frame after frame, with the two exchanges ----
    cudaEvent_t t1b = nullptr, t2 = nullptr;
    if (m->timing) { t1b = ev_get(m); t2 = ev_get(m); cudaEventRecord(t1b, st); }
    const int grid = m->nsm;
    for (int i = 0; i < Wn; ++i) {
      for (int l = 0; l < L; ++l) {
        disc_map* s = Gp.sh[l];
        launch_stage2_sharded_frame(0, i, Gp.meta, s->Wb[1], s->M, s->X, s->P, sem, grid, st);
        const int g = Gp.nccl ? Gp.rank : l;
        launch_trip_pack(s->X, Gp.trip_all + (size_t)g * Gp.trip_stride, s->X.TCAP, s->d_err, st);
      }
      if (Gp.nccl) {
        const int rc = Gp.nc.all_gather(Gp.trip_all + (size_t)Gp.rank * Gp.trip_stride, Gp.trip_all, Gp.trip_stride,
                                        NcclApi::U32, Gp.comm, st);
        if (rc) return group_fail_nccl(m, rc, "ncclAllGather(triples)");
      }
      for (int l = 0; l < L; ++l) {
        disc_map* s = Gp.sh[l];
        launch_trip_merge(s->X, Gp.trip_all, Gp.trip_stride, G, Gp.nccl ? Gp.rank : l, s->d_err, st);
        launch_stage2_sharded_frame(1, i, Gp.meta, s->Wb[1], s->M, s->X, s->P, sem, grid, st);
        launch_stage2_sharded_frame(2, i, Gp.meta, s->Wb[1], s->M, s->X, s->P, sem, grid, st);
        launch_add_pack(s->M, s->X, Gp.add_all + (size_t)(Gp.nccl ? 0 : l) * Gp.add_stride, SM, st);
      }
      int parts = G;
      if (Gp.nccl) {
        const int rc = Gp.nc.all_reduce(Gp.add_all, Gp.add_all, Gp.add_stride, NcclApi::I64, NcclApi::SUM, Gp.comm, st);
        if (rc) return group_fail_nccl(m, rc, "ncclAllReduce(new memberships)");
        parts = 1;
      }
      for (int l = 0; l < L; ++l)
        launch_finalize_sum(i, Gp.sh[l]->M, Gp.sh[l]->X, Gp.add_all, parts, Gp.add_stride, SM, st);
      m->stats.launches += 5 * L;
    }
    if (t2) {
      cudaEventRecord(t2, st);
      m->ev_pending.push_back({t1b, t2, 2});
    }
    m->stats.frames += Wn;
    disc_status cs = cuda_check(m, "sharded integrate launch");
    if (cs != DISC_OK) return cs;
    // last-frame bookkeeping of every local shard (debug export)
    cudaMemcpyAsync(Gp.h_meta, Gp.meta, sizeof(FrameMeta) * Wn, cudaMemcpyDeviceToHost, st);
    if (reports) cudaMemcpyAsync(Gp.h_rep, Gp.sh[0]->X.rep, sizeof(disc_frame_report) * Wn, cudaMemcpyDeviceToHost, st);
    const disc_status ss = group_sync(m, st);
    if (ss != DISC_OK) return ss;
    if (reports)
      for (int j = 0; j < nc; ++j) reports[w0 + j] = Gp.h_rep[Gp.nccl ? Gp.rank + G * j : j];
    for (disc_map* s : Gp.sh) {
      s->have_last = true;
      s->last_buf = 1;
      s->last_f = Wn - 1;
      s->last_fd = FrameDesc{};
      s->last_fd.S = Gp.h_meta[Wn - 1].S;
      s->last_stream = st;
    }
  }
  cudaEventRecord(m->ev_done, st);   // disc_wait orders other streams after the map's work
  return cuda_check(m, "sharded integrate");
}

// SMs for stage 2 in the next window: the base split plus, when the stream's frames carry many
// (mask, voxel) pairs (far views, H-shaped maps), more SMs for the lookup / apply work that grows
// with them (measured: H-shaped 108 k pairs per frame, 20 -> 64 SMs: +42 % frames/s; R-shaped 20 k: no
// gain).  The level comes from pair counts already copied back, never from a wait.
static int stage2_reserve(disc_map* m, bool sem) {
  for (int bb = 0; bb < 2; ++bb) {
    if (!m->np_pending[bb]) continue;
    const cudaError_t q = cudaEventQuery(m->ev_np[bb]);
    if (q == cudaSuccess) {
      uint64_t sum = 0;
      for (int i = 0; i < m->np_pending[bb]; ++i) sum += m->h_np[(size_t)bb * MAXWIN + i];
      m->np_avg = (double)sum / m->np_pending[bb];
      m->np_pending[bb] = 0;
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();   // (not an error)
    }
  }
  const int base = sem ? m->nres : m->nres_geo;
  int extra = 0;
  // one more SM per 1 k pairs above 24 k per frame, up to 100 SMs for geometry-only windows and 80 for
  // CLIP windows (final round-2 build, H, two runs each: 100/80 M1 16.9/16.8 k, M2 12.3/12.3 k;
  // 108/88 16.5/16.6 k, 12.2/12.2 k; 116/96 16.0/16.4 k, 11.8/11.7 k); earlier builds, measured
  // on the prefilled H map, 85 k pairs per frame: 74 SMs 13.8 k, 104 SMs 14.5 k frames/s; at ~110
  // stage 1 turns critical) and 88 for windows with CLIP tokens (H M2, round 2 with stage 1 kept off
  // stage 2's SMs: 56 SMs 9.5 k, 72 10.3 k, 80 10.7 k, 88 10.75 k frames/s, stage 1 then 2.4 ms/window)
  if (m->adapt && base > 0 && m->np_avg > 24000.0)
    extra = (int)std::min(sem ? 54.0 : 52.0, (m->np_avg - 24000.0) / 1000.0);
  return std::min(base + extra, m->nsm * 3 / 4);
}

// host-input staging: one window of frames' inputs (pinned host -> device, stream-ordered)
static disc_status ensure_stage(disc_map* m) {
  if (m->stage_buf[0]) return DISC_OK;
  const disc_config& c = m->cfg;
  m->stage_bytes = (size_t)c.window * ((size_t)c.max_pixels * (4 + c.max_masks) + (size_t)c.max_masks * 4 + 256 +
                                       (size_t)c.max_patches * ((size_t)c.feat_dim * 4 + (size_t)c.track_dim * 2) +
                                       (size_t)c.feat_dim * 4 + 4096);
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc((void**)&m->stage_buf[i], m->stage_bytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->ev_stage[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&m->ev_h2d[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return fail(m, DISC_ERR_CAPACITY, "cannot allocate host-input staging buffers");
    }
  }
  if (cudaStreamCreateWithFlags(&m->s0, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return fail(m, DISC_ERR_CUDA, "cannot create the host-input copy stream");
  }
  m->stage = m->stage_buf[0];
  return DISC_OK;
}

static void stage_frame(disc_map* m, size_t& so, disc_frame& f, cudaStream_t st) {
  const int Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  auto put = [&](const void* src, size_t bytes) -> const void* {
    if (!src || !bytes) return nullptr;
    so = (so + 255) & ~(size_t)255;
    void* dst = m->stage + so;
    cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    so += bytes;
    return dst;
  };
  const size_t HW = (size_t)f.height * f.width, Pn = (size_t)f.patch_h * f.patch_w;
  f.depth = (const float*)put(f.depth, HW * 4);
  f.masks = (const uint8_t*)put(f.masks, HW * f.num_masks);
  f.mask_bits = (const uint32_t*)put(f.mask_bits, (HW + 31) / 32 * 4 * f.num_masks);
  f.mask_conf = (const float*)put(f.mask_conf, (size_t)f.num_masks * 4);
  f.patch_feats = (const float*)put(f.patch_feats, Pn * Df * 4);
  f.global_embed = (const float*)put(f.global_embed, (size_t)Df * 4);
  f.track_feats = (const uint16_t*)put(f.track_feats, Dt > 0 ? Pn * Dt * 2 : 0);
}

static disc_status integrate_impl(disc_map* m, const disc_frame* frames, int32_t n, void* stream,
                                  disc_frame_report* reports, bool host_inputs) {
  if (!m || (!frames && n > 0) || n < 0) return DISC_ERR_INVALID;
  if (m->sticky != DISC_OK) return m->sticky;
  cudaSetDevice(m->dev);
  cudaStream_t st = (cudaStream_t)stream;
  m->last_stream = st;
  // O0: validate every frame before any mutation
  for (int i = 0; i < n; ++i) {
    const std::string v = validate_frame(m, frames[i], host_inputs);
    if (!v.empty()) return fail(m, DISC_ERR_INVALID, "frame " + std::to_string(i) + ": " + v);
  }
  const disc_config& c = m->cfg;
  const int win = c.window;
  const int Df = c.feat_dim, Dt = c.track_dim;
  if (host_inputs) {
    const disc_status ss = ensure_stage(m);
    if (ss != DISC_OK) return ss;
    if (reports && m->h_rep_cap < n) {
      if (m->h_rep_all) cudaFreeHost(m->h_rep_all);
      m->h_rep_all = nullptr;
      m->h_rep_cap = 0;
      if (cudaMallocHost(&m->h_rep_all, sizeof(disc_frame_report) * (size_t)std::max(n, 64)) != cudaSuccess) {
        cudaGetLastError();
        return fail(m, DISC_ERR_CAPACITY, "cannot allocate pinned report buffer");
      }
      m->h_rep_cap = std::max(n, 64);
    }
  }
  // stream-ordered after the caller's prior work on `st`; stage 1 on s1, stage 2 on s2
  cudaEventRecord(m->ev_in, st);
  cudaStreamWaitEvent(m->s1, m->ev_in, 0);
  cudaStreamWaitEvent(m->s2, m->ev_in, 0);
  if (host_inputs) cudaStreamWaitEvent(m->s0, m->ev_in, 0);
  cudaStream_t s1 = m->s1, s2 = m->s2;
  for (int w0 = 0; w0 < n; w0 += win) {
    const int nw = std::min(win, n - w0);
    const int b = m->wbuf;
    m->wbuf ^= 1;
    WinBufs& Wbuf = m->Wb[b];
    if (m->s2_pending[b]) cudaStreamWaitEvent(s1, m->ev_s2[b], 0);   // stage 2 done with this buffer
    WinDesc wd{};
    wd.n = nw;
    wd.Df = Df;
    wd.Dt = Dt;
    int maxS = 1, maxHp = 1, maxW = 1, maxWp = 1, maxP = 1, rows = 4;
    bool sem = false;
    size_t so = 0;
    int sb = 0;
    if (host_inputs) {   // the staging buffer stage 1 of the window before last has finished reading
      sb = m->stage_next;
      m->stage_next ^= 1;
      if (m->stage_pending[sb]) cudaStreamWaitEvent(m->s0, m->ev_stage[sb], 0);
      m->stage = m->stage_buf[sb];
    }
    for (int i = 0; i < nw; ++i) {
      disc_frame f = frames[w0 + i];
      // this frame's inputs to device staging, on the copy stream: window w+1's copies run beside
      // window w's stage 1 and stage 2 (two staging buffers), stage 1 waits for its own
      if (host_inputs) stage_frame(m, so, f, m->s0);
      wd.f[i] = make_desc(f);
      maxS = std::max(maxS, f.num_masks);
      maxHp = std::max(maxHp, f.patch_h);
      maxW = std::max(maxW, f.width);
      maxWp = std::max(maxWp, f.patch_w);
      maxP = std::max(maxP, f.patch_h * f.patch_w);
      sem = sem || f.patch_feats != nullptr;
      m->stats.mask_bytes += (int64_t)f.height * f.width * f.num_masks;
      m->stats.depth_bytes += (int64_t)f.height * f.width * 4;
      m->stats.track_bytes += (int64_t)f.patch_h * f.patch_w * Dt * 2;
      if (f.patch_feats) m->stats.feat_bytes += (int64_t)f.patch_h * f.patch_w * Df * 4;
    }
    if (host_inputs) {
      cudaEventRecord(m->ev_h2d[sb], m->s0);
      cudaStreamWaitEvent(s1, m->ev_h2d[sb], 0);
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr, t0 = nullptr, t1 = nullptr, t1b = nullptr, t2 = nullptr;
    if (m->timing) {
      e0 = ev_get(m); e1 = ev_get(m); t0 = ev_get(m); t1 = ev_get(m); t1b = ev_get(m); t2 = ev_get(m);
      cudaEventRecord(t0, s1);
    }
    tl_mark(s1, "s1_begin", -1);
    const int nres_w = stage2_reserve(m, sem);
    // frame tables: fill the dirty ones; release after use when they are much larger than a frame's pairs
    const bool release = m->np_avg > 0.0 && (double)Wbuf.PC > m->tab_ratio * m->np_avg;
    m->stats.launches += launch_stage1(wd, Wbuf, m->P, m->d_err, sem, maxS, maxHp, maxW, maxWp, maxP, rows, m->nsm,
                                       nres_w, s1, e0, e1, !m->ktab_clean[b], !m->nsum_clean[b], release);
    m->ktab_clean[b] = release;
    if (sem) m->nsum_clean[b] = release;
    if (host_inputs) {
      cudaEventRecord(m->ev_stage[sb], s1);
      m->stage_pending[sb] = true;
    }
    cudaMemcpyAsync(m->h_np + (size_t)b * MAXWIN, Wbuf.npairs, sizeof(uint32_t) * nw, cudaMemcpyDeviceToHost, s1);
    cudaEventRecord(m->ev_np[b], s1);
    m->np_pending[b] = nw;
    if (m->timing) cudaEventRecord(t1, s1);
    cudaEventRecord(m->ev_s1[b], s1);
    cudaStreamWaitEvent(s2, m->ev_s1[b], 0);
    if (m->timing) cudaEventRecord(t1b, s2);
    tl_mark(s2, "s2_begin", -1);
    m->stats.launches += launch_stage2(wd, Wbuf, m->M, m->X, m->P, sem, m->nsm, nres_w, &m->s2_tag, m->s2_spec, s2);
    if (m->timing) {
      cudaEventRecord(t2, s2);
      m->ev_pending.push_back({e0, e1, 0});
      m->ev_pending.push_back({t0, t1, 1});
      m->ev_pending.push_back({t1b, t2, 2});
    }
    cudaEventRecord(m->ev_s2[b], s2);
    m->s2_pending[b] = true;
    m->stats.frames += nw;
    disc_status cs = cuda_check(m, "integrate launch");
    if (cs != DISC_OK) return cs;
    if (reports && host_inputs) {   // (stream-ordered before the next window's stage 2 rewrites X.rep)
      cudaMemcpyAsync(m->h_rep_all + w0, m->X.rep, sizeof(disc_frame_report) * nw, cudaMemcpyDeviceToHost, s2);
    } else if (reports) {
      cudaMemcpyAsync(m->h_rep, m->X.rep, sizeof(disc_frame_report) * nw, cudaMemcpyDeviceToHost, s2);
      disc_status ss = sync_check(m, s2);
      if (ss != DISC_OK) return ss;
      std::memcpy(reports + w0, m->h_rep, sizeof(disc_frame_report) * nw);
    }
    m->have_last = true;
    m->last_buf = b;
    m->last_f = nw - 1;
    m->last_fd = wd.f[nw - 1];
    m->last_sem = sem;
  }
  // the caller's stream is ordered after stage 1 (the last reader of the caller's inputs);
  // stage 2 may still run on s2: disc_wait / disc_sync / every reader order after it
  cudaEventRecord(m->ev_done, s2);
  cudaEventRecord(m->ev_s1done, s1);
  cudaStreamWaitEvent(st, m->ev_s1done, 0);
  if (host_inputs) {   // the caller's host buffers are free again on return; reports complete
    disc_status ss = sync_check(m, reports ? s2 : st);
    if (ss != DISC_OK) return ss;
    if (reports) std::memcpy(reports, m->h_rep_all, sizeof(disc_frame_report) * n);
  }
  return cuda_check(m, "integrate launch");
}

disc_status disc_integrate_frame(disc_map* m, const disc_frame* f, void* stream, disc_frame_report* report) {
  if (m && m->grp) return group_integrate(m, f, 1, stream, report, false);
  return integrate_impl(m, f, 1, stream, report, false);
}

disc_status disc_integrate_frames(disc_map* m, const disc_frame* f, int32_t n, void* stream,
                                  disc_frame_report* report) {
  if (m && m->grp) return group_integrate(m, f, n, stream, report, false);
  return integrate_impl(m, f, n, stream, report, false);
}

disc_status disc_integrate_frames_host(disc_map* m, const disc_frame* f, int32_t n, void* stream,
                                       disc_frame_report* report) {
  if (!m || (!f && n > 0) || n < 0) return DISC_ERR_INVALID;
  if (m->grp) return group_integrate(m, f, n, stream, report, true);
  if (m->sticky != DISC_OK) return m->sticky;
  // O0 over ALL n frames before the first window mutates the map (disc.h: INVALID = nothing changed)
  for (int i = 0; i < n; ++i) {
    const std::string v = validate_frame(m, f[i], true);
    if (!v.empty()) return fail(m, DISC_ERR_INVALID, "frame " + std::to_string(i) + ": " + v);
  }
  // windows pipelined over two staging buffers; one synchronisation at the end of the call
  return integrate_impl(m, f, n, stream, report, true);
}

static disc_status ensure_scratch(disc_map* m, size_t bytes) {
  if (m->scratch_bytes >= bytes) return DISC_OK;
  if (m->scratch) cudaFree(m->scratch);
  m->scratch = nullptr;
  m->scratch_bytes = 0;
  if (cudaMalloc(&m->scratch, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(m, DISC_ERR_CAPACITY, "cannot allocate export scratch");
  }
  m->scratch_bytes = bytes;
  return DISC_OK;
}

static int64_t host_next_id(disc_map* m) {
  int64_t nid = 0;
  cudaMemcpy(&nid, m->M.counters, sizeof(int64_t), cudaMemcpyDeviceToHost);
  return nid;
}

disc_status disc_wait(disc_map* m, void* stream) {
  if (!m) return DISC_ERR_INVALID;
  if (m->sticky != DISC_OK) return m->sticky;
  cudaSetDevice(m->dev);
  cudaStreamWaitEvent((cudaStream_t)stream, m->ev_done, 0);
  return cuda_check(m, "disc_wait");
}

disc_status disc_sync(disc_map* m) {
  if (!m) return DISC_ERR_INVALID;
  if (m->sticky != DISC_OK) return m->sticky;
  cudaSetDevice(m->dev);
  if (m->grp) return group_sync(m, m->last_stream);
  if (m->s1) cudaStreamSynchronize(m->s1);
  if (m->s2) cudaStreamSynchronize(m->s2);
  tl_dump();
  return sync_check(m, m->last_stream);
}

disc_status disc_query(disc_map* m, const float* q, int32_t k, int64_t* ids, float* scores, int32_t* n_out) {
  if (!m || !q || k < 0 || (k > 0 && (!ids || !scores)) || !n_out) return DISC_ERR_INVALID;
  if (m->grp) {   // the instance table is replicated: shard 0 answers
    const disc_status gs = disc_sync(m);
    return gs != DISC_OK ? gs : disc_query(m->grp->sh[0], q, k, ids, scores, n_out);
  }
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  const int64_t nid = host_next_id(m);
  const size_t need = (size_t)(nid + 16) * 24 + (size_t)m->cfg.feat_dim * 4 + (16 << 20);
  if ((s = ensure_scratch(m, need)) != DISC_OK) return s;
  const int32_t r = run_query(m->M, m->cfg.feat_dim, nid, q, k, ids, scores, m->last_stream, m->scratch, m->scratch_bytes);
  if (r < 0) return fail(m, DISC_ERR_INTERNAL, "query scratch too small");
  *n_out = r;
  return cuda_check(m, "disc_query");
}

disc_status disc_get_instances(disc_map* m, disc_instance* out, float* embeds, double* track, int32_t cap,
                               int32_t* n_out) {
  if (!m || !n_out) return DISC_ERR_INVALID;
  if (m->grp) {   // replicated instance table (|V| summed over the shards' keys every frame)
    const disc_status gs = disc_sync(m);
    return gs != DISC_OK ? gs : disc_get_instances(m->grp->sh[0], out, embeds, track, cap, n_out);
  }
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  const int64_t nid = host_next_id(m);
  const int Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  const size_t per = sizeof(disc_instance) + (size_t)Df * 4 + (size_t)std::max(Dt, 1) * 8 + 16;
  const size_t need = (size_t)(nid + 16) * (8 + per) + (16 << 20);
  if ((s = ensure_scratch(m, need)) != DISC_OK) return s;
  const int64_t n = export_instances(m->M, Df, Dt, nid, out, embeds, track, out ? cap : 0, m->last_stream,
                                     m->scratch, m->scratch_bytes);
  if (n < 0) return fail(m, DISC_ERR_INTERNAL, "export scratch too small");
  *n_out = (int32_t)n;
  if (out && n > cap) return fail(m, DISC_ERR_INVALID, "cap too small");
  return cuda_check(m, "disc_get_instances");
}

disc_status disc_get_memberships(disc_map* m, uint64_t* keys, int64_t* ids, int64_t cap, int64_t* n_out) {
  if (!m || !n_out || (keys && !ids)) return DISC_ERR_INVALID;
  if (m->grp) {   // the shards' key sets are disjoint: the union is their concatenation (this process's shards)
    disc_status gs = disc_sync(m);
    if (gs != DISC_OK) return gs;
    int64_t tot = 0;
    for (disc_map* sh : m->grp->sh) {
      int64_t k = 0;
      gs = disc_get_memberships(sh, keys ? keys + tot : nullptr, keys ? ids + tot : nullptr,
                                keys ? std::max<int64_t>(0, cap - tot) : 0, &k);
      if (gs != DISC_OK) return fail(m, gs, sh->err);
      tot += k;
    }
    *n_out = tot;
    return DISC_OK;
  }
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  const size_t need = (size_t)(keys ? cap : 0) * 16 + (1 << 20);
  if ((s = ensure_scratch(m, need)) != DISC_OK) return s;
  const int64_t n = export_memberships(m->M, keys, ids, keys ? cap : 0, m->last_stream, m->scratch, m->scratch_bytes);
  if (n < 0) return fail(m, DISC_ERR_INTERNAL, "export scratch too small");
  *n_out = n;
  if (keys && n > cap) return fail(m, DISC_ERR_INVALID, "cap too small");
  return cuda_check(m, "disc_get_memberships");
}

disc_status disc_debug_last_frame(disc_map* m, disc_frame_debug* d) {
  if (!m || !d) return DISC_ERR_INVALID;
  if (m->grp) {   // replicated records and (merged) triples; each shard's share of the pairs
    disc_status gs = disc_sync(m);
    if (gs != DISC_OK) return gs;
    int64_t k = 0;
    for (disc_map* sh : m->grp->sh) {
      disc_frame_debug dl = *d;
      if (d->pair_s) {
        dl.pair_s = d->pair_s + std::min(k, d->pair_cap);
        dl.pair_key = d->pair_key + std::min(k, d->pair_cap);
        dl.pair_cap = std::max<int64_t>(0, d->pair_cap - k);
      }
      gs = disc_debug_last_frame(sh, &dl);
      if (gs != DISC_OK) return fail(m, gs, sh->err);
      k += dl.n_pairs;
      d->num_masks = dl.num_masks;
      d->n_trip = dl.n_trip;
    }
    d->n_pairs = k;
    return DISC_OK;
  }
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  if (!m->have_last) return fail(m, DISC_ERR_INVALID, "no frame integrated yet");
  const int S = m->last_fd.S, f = m->last_f, SM = m->cfg.max_masks, Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  const WinBufs& W = m->Wb[m->last_buf];
  d->num_masks = S;
  const size_t fo = (size_t)f * SM;
  std::vector<int32_t> status(S);
  cudaMemcpy(status.data(), W.status + fo, 4 * S, cudaMemcpyDeviceToHost);
  if (d->status) std::memcpy(d->status, status.data(), 4 * S);
  if (d->area) {
    std::vector<uint32_t> a(S);
    cudaMemcpy(a.data(), W.area + fo, 4 * S, cudaMemcpyDeviceToHost);
    for (int i = 0; i < S; ++i) d->area[i] = a[i];
  }
  if (d->bbox) cudaMemcpy(d->bbox, W.bbox + 4 * fo, 16 * S, cudaMemcpyDeviceToHost);
  if (d->vs) {
    std::vector<uint32_t> a(S);
    cudaMemcpy(a.data(), W.vs + fo, 4 * S, cudaMemcpyDeviceToHost);
    for (int i = 0; i < S; ++i) d->vs[i] = a[i];
  }
  if (d->target) cudaMemcpy(d->target, m->X.det_id, 8 * S, cudaMemcpyDeviceToHost);
  if (d->factors) cudaMemcpy(d->factors, W.qf + 6 * fo, 24 * S, cudaMemcpyDeviceToHost);
  if (d->embed) cudaMemcpy(d->embed, W.emb + fo * Df, (size_t)4 * S * Df, cudaMemcpyDeviceToHost);
  if (d->track && Dt > 0) cudaMemcpy(d->track, W.trk + fo * Dt, (size_t)8 * S * Dt, cudaMemcpyDeviceToHost);
  // pairs of kept detections
  uint32_t np = 0;
  cudaMemcpy(&np, W.npairs + f, 4, cudaMemcpyDeviceToHost);
  np = std::min<uint32_t>(np, (uint32_t)W.PMAX);
  std::vector<unsigned long long> pk(np);
  std::vector<uint32_t> ps(np);
  cudaMemcpy(pk.data(), W.pkey + (size_t)f * W.PMAX, 8ull * np, cudaMemcpyDeviceToHost);
  cudaMemcpy(ps.data(), W.pinfo + (size_t)f * W.PMAX, 4ull * np, cudaMemcpyDeviceToHost);
  int64_t k = 0;
  for (uint32_t i = 0; i < np; ++i) {
    if (ps[i] >= (uint32_t)S || status[ps[i]] != 0) continue;
    if (d->pair_s && k < d->pair_cap) {
      d->pair_s[k] = (int32_t)ps[i];
      d->pair_key[k] = pk[i];
    }
    k++;
  }
  d->n_pairs = k;
  uint32_t nt = 0;
  cudaMemcpy(&nt, m->X.ntrip_last, 4, cudaMemcpyDeviceToHost);
  nt = std::min<uint32_t>(nt, (uint32_t)m->X.TCAP);
  std::vector<uint32_t> ts(nt), tj(nt), tc(nt);
  std::vector<uint8_t> te(nt);
  cudaMemcpy(ts.data(), m->X.trip_sd, 4ull * nt, cudaMemcpyDeviceToHost);
  cudaMemcpy(tj.data(), m->X.trip_jd, 4ull * nt, cudaMemcpyDeviceToHost);
  cudaMemcpy(tc.data(), m->X.trip_c, 4ull * nt, cudaMemcpyDeviceToHost);
  cudaMemcpy(te.data(), m->X.trip_edge, 1ull * nt, cudaMemcpyDeviceToHost);
  // a speculatively counted frame's table can hold (s, label) entries whose count its predecessor's
  // update took back to 0 (a merged-away label): not triples of C
  uint32_t kt = 0;
  for (uint32_t i = 0; i < nt; ++i) {
    if (tc[i] == 0) continue;
    if (d->trip_s && kt < (uint32_t)d->trip_cap) {
      d->trip_s[kt] = (int32_t)ts[i];
      d->trip_j[kt] = tj[i];
      d->trip_c[kt] = tc[i];
      d->trip_edge[kt] = te[i];
    }
    kt++;
  }
  d->n_trip = kt;
  return cuda_check(m, "disc_debug_last_frame");
}

disc_status disc_classify(disc_map* m, const float* table, int32_t C, int32_t k, int64_t* ids, int32_t* classes,
                          float* scores, int64_t cap, int64_t* n_out) {
  if (!m || !table || C < 1 || k < 1 || k > 16 || !n_out || cap < 0 || (ids && (!classes || !scores)))
    return DISC_ERR_INVALID;
  if (m->grp) {   // the instance table (and its embeddings) is replicated: shard 0 answers
    const disc_status gs = disc_sync(m);
    return gs != DISC_OK ? gs : disc_classify(m->grp->sh[0], table, C, k, ids, classes, scores, cap, n_out);
  }
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  const int64_t nid = host_next_id(m);
  const int kk = std::min(k, C);
  const size_t need = (size_t)(nid + 16) * (16 + 8 * (size_t)kk) + (size_t)C * (m->cfg.feat_dim * 4 + 8) + (16 << 20);
  if ((s = ensure_scratch(m, need)) != DISC_OK) return s;
  const int64_t n = run_classify(m->M, m->cfg.feat_dim, nid, table, C, k, ids, classes, scores, ids ? cap : 0,
                                 m->last_stream, m->scratch, m->scratch_bytes);
  if (n < 0) return fail(m, DISC_ERR_INTERNAL, "classify scratch too small");
  *n_out = n;
  if (ids && n > cap) return fail(m, DISC_ERR_INVALID, "cap too small");
  return cuda_check(m, "disc_classify");
}

disc_status disc_dense_transfer(disc_map* m, const float* points, int64_t P, float d_assign, int64_t* out) {
  if (!m || P < 0 || (P > 0 && (!points || !out)) || !(d_assign >= 0.0f) || !std::isfinite(d_assign))
    return DISC_ERR_INVALID;
  if (m->grp) return fail(m, DISC_ERR_UNSUPPORTED, "disc_dense_transfer: sharded maps are not supported");
  if (d_assign / m->cfg.voxel_size > 64.0f) return fail(m, DISC_ERR_INVALID, "d_assign above 64 voxels");
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  if (P == 0) return DISC_OK;
  if ((s = ensure_scratch(m, (size_t)P * 20 + (1 << 20))) != DISC_OK) return s;
  if (run_dense_transfer(m->M, m->cfg.voxel_size, points, P, d_assign, out, m->last_stream, m->scratch,
                         m->scratch_bytes) != 0)
    return fail(m, DISC_ERR_INTERNAL, "dense transfer scratch too small");
  return cuda_check(m, "disc_dense_transfer");
}

disc_status disc_finalize(disc_map* m, float tau_geo, float tau_vis, int64_t min_voxels, disc_final_report* rep) {
  if (!m || !(tau_geo > 0.0f && tau_geo <= 1.0f) || !(tau_vis >= -1.0f && tau_vis <= 1.0f) || min_voxels < 0)
    return DISC_ERR_INVALID;
  if (m->grp) return fail(m, DISC_ERR_UNSUPPORTED, "disc_finalize: sharded maps are not supported");
  disc_status s = disc_sync(m);
  if (s != DISC_OK) return s;
  int64_t r[7] = {0, 0, 0, 0, 0, 0, 0};
  if (run_finalize(m->M, m->cfg.feat_dim, m->cfg.track_dim, host_next_id(m), tau_geo, tau_vis, min_voxels, m->d_err,
                   m->last_stream, r) != 0)
    return fail(m, DISC_ERR_CAPACITY, "disc_finalize: cannot allocate its temporary buffers");
  s = sync_check(m, m->last_stream);
  if (s != DISC_OK) return s;
  if (rep) {
    rep->rounds = r[0]; rep->edges = r[1]; rep->merged_away = r[2]; rep->relabeled = r[3]; rep->removed = r[4];
    rep->live_instances = r[5]; rep->live_memberships = r[6];
  }
  return cuda_check(m, "disc_finalize");
}

disc_status disc_set_timing(disc_map* m, int32_t on) {
  if (!m) return DISC_ERR_INVALID;
  m->timing = on != 0;
  return DISC_OK;
}

disc_status disc_get_stats(disc_map* m, disc_stats* s) {
  if (!m || !s) return DISC_ERR_INVALID;
  disc_status st = disc_sync(m);
  if (st != DISC_OK) return st;
  collect_events(m);
  if (m->grp) {   // U and edges are replicated; inserts / relabel items are per shard (own keys)
    m->stats.pairs = m->stats.map_inserts = m->stats.relabels = m->stats.edges = 0;
    for (size_t l = 0; l < m->grp->sh.size(); ++l) {
      int64_t ctr[8];
      cudaMemcpy(ctr, m->grp->sh[l]->M.counters, sizeof(ctr), cudaMemcpyDeviceToHost);
      if (l == 0) { m->stats.pairs = ctr[4]; m->stats.edges = ctr[7]; }
      m->stats.map_inserts += ctr[5];
      m->stats.relabels += ctr[6];
      if (l < 16) m->stats.shard_memberships[l] = ctr[2];   // own keys' live memberships
    }
    *s = m->stats;
    return cuda_check(m, "disc_get_stats");
  }
  if (getenv("DISC_K6PROF") || getenv("DISC_S2PROF")) k6_prof_dump();
  if (getenv("DISC_SLOT_STATS") && !m->grp) slot_stats(m->M, m->last_stream);
  int64_t ctr[8];
  cudaMemcpy(ctr, m->M.counters, sizeof(ctr), cudaMemcpyDeviceToHost);
  m->stats.pairs = ctr[4];
  m->stats.map_inserts = ctr[5];
  m->stats.relabels = ctr[6];
  m->stats.edges = ctr[7];
  m->stats.shard_memberships[0] = ctr[2];
  *s = m->stats;
  return cuda_check(m, "disc_get_stats");
}

const char* disc_last_error(const disc_map* m) { return m ? m->err.c_str() : "null map"; }

}  // extern "C"
