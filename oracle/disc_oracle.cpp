/*
 * disc_oracle.cpp -- plain, slow, definitional CPU oracle of the DISC per-frame mapping
 * hot path (arXiv 2603.03935, §III).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs; never by the product path.  It shares no code
 * with the CUDA path (paper_2603_03935_b200/csrc).
 *
 * Build: g++ -std=c++17 -O2 -ffp-contract=off (no fast-math): the pinned fp32 key formula
 * (R5) relies on IEEE single-precision '/', 'fmaf' and 'floorf' without contraction.
 *
 * State (C.1): std::map<Key, std::set<Id>> (membership relation, key -> ids) and
 * std::map<Id, Inst> (id -> voxel set + fused attributes); the two are cross-checked by
 * the self-check.  Floating point of the semantic part is fp64 (Eq.1-3); keys are pinned
 * fp32 (R5); the visual gate is pinned fp64 (R15).
 *
 * Pins: tests/test_oracle_pins.py (SPEC worked examples, the hand-worked T0 fixture,
 * brute force, closed forms, invariants).  Every function below names the passage it
 * follows.  Parity of S_angle normals follows reading R21 (paper silent).
 */
#include "disc_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <string>
#include <vector>

namespace {

using Key = std::array<int32_t, 3>;  // (ix, iy, iz) voxel grid indices
using Id = int64_t;
constexpr int32_t KEY_BIAS = 1 << 20;  // R6: components in [-2^20, 2^20)

uint64_t pack(const Key& k) {  // R6: 3 x 21-bit, biased; order-preserving
  return ((uint64_t)(uint32_t)(k[0] + KEY_BIAS) << 42) |
         ((uint64_t)(uint32_t)(k[1] + KEY_BIAS) << 21) | (uint64_t)(uint32_t)(k[2] + KEY_BIAS);
}

double bf16_to_double(uint16_t b) {  // bf16 = upper 16 bits of an IEEE fp32
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}

struct Obs {  // one fused observation (for the R22 acceptance set)
  double q;
  std::vector<double> e;
};

struct Inst {  // C.1 instance node
  std::set<Key> V;
  int32_t obs = 0;
  int64_t last_seen = 0;
  double Q = -1.0;            // -1 = no embedding observed yet (geometry-only mode)
  std::vector<double> e;      // unit vector [Df] (zeros while Q == -1)
  std::vector<double> T;      // fp64 sum of fused tracking features [Dt] (R15)
  std::vector<Obs> accept;    // observations with q >= qmax*(1-1e-4)   (R22)
};

struct Det {  // per-mask record of one frame
  int32_t status = ORA_KEPT;
  int64_t area = 0;
  int32_t bbox[4] = {0, 0, -1, -1};  // umin, vmin, umax, vmax
  std::set<Key> V;
  std::map<Key, std::array<double, 3>> nsum;  // O4: sum of pixel normals per voxel
  std::map<Key, int64_t> nnorm;               // number of pixel normals summed per voxel
  double f[6] = {0, 0, 0, 0, -1, 0};          // s_size, s_angle, s_sem, s_dist, q, dbar
  std::vector<double> e, u, t;
  bool t_ok = false;
  int64_t target = -1;
};

}  // namespace

struct ora_map {
  ora_config cfg;
  bool selfcheck = false;
  std::map<Key, std::set<Id>> mem;  // membership relation {(k, id)}
  std::map<Id, Inst> inst;
  Id next_id = 0;
  std::string err;
  // last-frame debug
  std::vector<Det> last;
  std::map<std::pair<int32_t, Id>, int64_t> last_c;
  std::set<std::pair<int32_t, Id>> last_edges;
};

/* ------------------------------------------------------------------------------------ */
/* single steps                                                                          */
/* ------------------------------------------------------------------------------------ */

extern "C" uint64_t ora_pack_key(int32_t ix, int32_t iy, int32_t iz) { return pack({ix, iy, iz}); }

/* A0: rotation orthonormal within 1e-5, det = +1 within 1e-5, last row 0 0 0 1. */
extern "C" int32_t ora_pose_rigid(const float* P) {
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(P[i])) return 0;
  if (P[12] != 0.0f || P[13] != 0.0f || P[14] != 0.0f || P[15] != 1.0f) return 0;
  double R[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = (double)P[4 * i + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = R[0][i] * R[0][j] + R[1][i] * R[1][j] + R[2][i] * R[2][j];  // (R^T R)_ij
      double want = (i == j) ? 1.0 : 0.0;
      if (std::fabs(s - want) > 1e-5) return 0;
    }
  double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
               R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
               R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  if (std::fabs(det - 1.0) > 1e-5) return 0;
  return 1;
}

/* O2, R1-R5 (S:117 p_w = R (d K^-1 [u,v,1]) + t): pinned fp32, no contraction. */
extern "C" int32_t ora_pixel_world(const ora_config* c, const ora_frame* f, int32_t u, int32_t v,
                                   float out[3]) {
  const float d = f->depth[(int64_t)v * f->width + u];
  if (!std::isfinite(d)) return 0;
  if (!(d > c->depth_min && d < c->depth_max)) return 0;  // R4 exclusive window
  const float a = (float)u - f->cx;
  const float xc = (a / f->fx) * d;
  const float b = (float)v - f->cy;
  const float yc = (b / f->fy) * d;
  const float zc = d;
  const float* M = f->pose;
  out[0] = std::fmaf(M[0], xc, std::fmaf(M[1], yc, std::fmaf(M[2], zc, M[3])));
  out[1] = std::fmaf(M[4], xc, std::fmaf(M[5], yc, std::fmaf(M[6], zc, M[7])));
  out[2] = std::fmaf(M[8], xc, std::fmaf(M[9], yc, std::fmaf(M[10], zc, M[11])));
  return 1;
}

/* O2, S:132-139 key = floor(p / r) (division, not multiplication by 1/r: R5); R6 range. */
extern "C" int32_t ora_point_key(const float p[3], float r, int32_t out[3]) {
  for (int i = 0; i < 3; ++i) {
    const float q = std::floor(p[i] / r);
    if (!(q >= -1048576.0f && q < 1048576.0f)) return 0;
    out[i] = (int32_t)q;
  }
  return 1;
}

/* Eq.1: D_p = |f_p - fbar| / (mean_p |f_p - fbar| + eps), fp64. */
extern "C" void ora_distinctiveness(int64_t P, int32_t Df, const float* F, double eps, double* D) {
  std::vector<double> fbar(Df, 0.0);
  for (int64_t p = 0; p < P; ++p)
    for (int32_t d = 0; d < Df; ++d) fbar[d] += (double)F[p * Df + d];
  for (int32_t d = 0; d < Df; ++d) fbar[d] /= (double)P;
  std::vector<double> r(P);
  double rsum = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double s = 0.0;
    for (int32_t d = 0; d < Df; ++d) {
      const double x = (double)F[p * Df + d] - fbar[d];
      s += x * x;
    }
    r[p] = std::sqrt(s);
    rsum += r[p];
  }
  const double rbar = rsum / (double)P;
  for (int64_t p = 0; p < P; ++p) D[p] = r[p] / (rbar + eps);
}

/* O7 pooling ("aggregating the patch features within the segmentation mask, weighted
 * by D"; R17-R19):
 *   w_p = D_p * cnt_p / npix_p  if cnt_p >= cover_min * npix_p (exact), else 0
 *   all w == 0 -> w_p = [cnt_p > 0]
 *   y = sum_p w_p f_p ; y == 0 -> "nofeat" ; e = y / |y|
 *   dbar = sum_{cnt>0} (cnt/npix) D / sum_{cnt>0} (cnt/npix)                  (R19) */
extern "C" int32_t ora_pool(int64_t P, int32_t Df, const int64_t* cnt, const int64_t* npix,
                            const double* D, const float* F, double cover_min, double* e,
                            double* dbar) {
  std::vector<double> w(P, 0.0);
  double wsum = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    if (cnt[p] > 0 && (double)cnt[p] >= cover_min * (double)npix[p]) {
      w[p] = D[p] * (double)cnt[p] / (double)npix[p];
      wsum += w[p];
    }
  }
  if (wsum == 0.0)
    for (int64_t p = 0; p < P; ++p) w[p] = cnt[p] > 0 ? 1.0 : 0.0;
  std::vector<double> y(Df, 0.0);
  for (int64_t p = 0; p < P; ++p)
    if (w[p] != 0.0)
      for (int32_t d = 0; d < Df; ++d) y[d] += w[p] * (double)F[p * Df + d];
  double nn = 0.0;
  for (int32_t d = 0; d < Df; ++d) nn += y[d] * y[d];
  double num = 0.0, den = 0.0;
  for (int64_t p = 0; p < P; ++p)
    if (cnt[p] > 0) {
      const double cov = (double)cnt[p] / (double)npix[p];
      num += cov * D[p];
      den += cov;
    }
  *dbar = den > 0.0 ? num / den : 0.0;
  if (nn == 0.0) {
    for (int32_t d = 0; d < Df; ++d) e[d] = 0.0;
    return 1;
  }
  const double n = std::sqrt(nn);
  for (int32_t d = 0; d < Df; ++d) e[d] = y[d] / n;
  return 0;
}

/* S_size = min(lambda |M| / (H W), 1) */
extern "C" double ora_s_size(int64_t area, int32_t H, int32_t W, double lambda) {
  return std::min(lambda * (double)area / ((double)H * (double)W), 1.0);
}

/* Eq.3: S_angle = (1/|V|) sum_v max(0, -r_v . n_v) */
extern "C" double ora_s_angle(int64_t n, const double* N, const double* Rr) {
  if (n <= 0) return 0.0;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double dot = Rr[3 * i] * N[3 * i] + Rr[3 * i + 1] * N[3 * i + 1] + Rr[3 * i + 2] * N[3 * i + 2];
    s += std::max(0.0, -dot);
  }
  return s / (double)n;
}

/* P:140, R20: S_sem = clamp(cos(e, g), 0, 1); g == NULL -> 1 */
extern "C" double ora_s_sem(int32_t Df, const double* e, const float* g) {
  if (!g) return 1.0;
  double dot = 0.0, gg = 0.0, ee = 0.0;
  for (int32_t d = 0; d < Df; ++d) {
    dot += e[d] * (double)g[d];
    gg += (double)g[d] * (double)g[d];
    ee += e[d] * e[d];
  }
  if (gg == 0.0 || ee == 0.0) return 0.0;
  const double c = dot / (std::sqrt(gg) * std::sqrt(ee));
  return std::min(std::max(c, 0.0), 1.0);
}

/* S_dist = 0.5 + 0.5 Dbar (unclamped above 1) */
extern "C" double ora_s_dist(double dbar) { return 0.5 + 0.5 * dbar; }

/* Eq.2: Q = S_geo S_sem S_dist, S_geo = S_size S_angle */
extern "C" double ora_quality(double s_size, double s_angle, double s_sem, double s_dist) {
  return ((s_size * s_angle) * s_sem) * s_dist;
}

/* R15: pinned fp64 dot.  Lane l (0..31) accumulates d = l, l+32, ... ascending with fma;
 * then the xor butterfly v_l <- v_l + v_{l^m} for m = 16, 8, 4, 2, 1; result = v_0. */
extern "C" double ora_dot_pin(int32_t n, const double* a, const double* b) {
  double lane[32];
  for (int l = 0; l < 32; ++l) {
    double acc = 0.0;
    for (int32_t d = l; d < n; d += 32) acc = std::fma(a[d], b[d], acc);
    lane[l] = acc;
  }
  for (int m = 16; m >= 1; m >>= 1) {
    double nxt[32];
    for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ m];
    std::memcpy(lane, nxt, sizeof(lane));
  }
  return lane[0];
}

/* P:92 [§III-A] "filtered using a custom, parallelized CUDA implementation of the DBSCAN algorithm
 * to remove noise"; "output labels equal those of the classic sequential DBSCAN".  The
 * classic algorithm (Ester et al. 1996) written out: points visited in index order; an unvisited
 * point with >= min_pts points within eps (itself included) starts a new cluster, which is expanded
 * breadth-first through core points; non-core points reached get the cluster (once) -- a border
 * point thus belongs to the first cluster that reaches it; the rest is noise.  R42: squared fp64
 * distance of the fp32 points, summed x, y, z, compared with (double)eps^2. */
extern "C" int32_t ora_dbscan(int64_t n, const float* pts, float eps, int32_t min_pts, int32_t* labels) {
  const double e2 = (double)eps * (double)eps;
  auto d2 = [&](int64_t a, int64_t b) {
    double s = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double x = (double)pts[3 * a + k] - (double)pts[3 * b + k];
      s = s + x * x;
    }
    return s;
  };
  auto neigh = [&](int64_t a) {
    std::vector<int64_t> out;
    for (int64_t b = 0; b < n; ++b)
      if (d2(a, b) <= e2) out.push_back(b);
    return out;
  };
  constexpr int32_t UNSEEN = -2, NOISE = -1;
  for (int64_t i = 0; i < n; ++i) labels[i] = UNSEEN;
  int32_t C = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (labels[i] != UNSEEN) continue;
    std::vector<int64_t> N = neigh(i);
    if ((int64_t)N.size() < min_pts) { labels[i] = NOISE; continue; }
    const int32_t c = C++;
    labels[i] = c;
    std::deque<int64_t> q(N.begin(), N.end());
    while (!q.empty()) {
      const int64_t j = q.front();
      q.pop_front();
      if (labels[j] == NOISE) labels[j] = c;   // border point (or a core point seen as noise earlier: impossible)
      if (labels[j] != UNSEEN) continue;
      labels[j] = c;
      std::vector<int64_t> Nj = neigh(j);
      if ((int64_t)Nj.size() >= min_pts) q.insert(q.end(), Nj.begin(), Nj.end());
    }
  }
  return C;
}

/* ------------------------------------------------------------------------------------ */
/* map                                                                                   */
/* ------------------------------------------------------------------------------------ */

static bool valid_config(const ora_config* c) {
  if (!c) return false;
  if (!(c->voxel_size > 0.0f) || !std::isfinite(c->voxel_size)) return false;
  if (!(c->tau_geo > 0.0f && c->tau_geo <= 1.0f)) return false;
  if (!(c->tau_vis >= -1.0f && c->tau_vis <= 1.0f)) return false;
  if (!(c->depth_min >= 0.0f && c->depth_min < c->depth_max)) return false;
  if (!(c->mask_min_conf >= 0.0f && c->mask_min_conf <= 1.0f)) return false;
  if (!(c->mask_max_aspect >= 1.0f) || c->mask_min_area < 0) return false;
  if (!(c->cover_min >= 0.0f && c->cover_min <= 1.0f)) return false;
  if (!(c->lambda_size > 0.0f) || !(c->eps_distinct >= 0.0f)) return false;
  if (!(c->dbscan_eps >= 0.0f) || (c->dbscan_eps > 0.0f && c->dbscan_min_pts < 1)) return false;
  if (c->feat_dim <= 0 || c->track_dim < 0) return false;
  return true;
}

extern "C" ora_map* ora_create(const ora_config* cfg) {
  if (!valid_config(cfg)) return nullptr;
  ora_map* m = new ora_map();
  m->cfg = *cfg;
  return m;
}
extern "C" void ora_destroy(ora_map* m) { delete m; }
extern "C" void ora_set_selfcheck(ora_map* m, int32_t on) { m->selfcheck = on != 0; }
extern "C" const char* ora_last_error(const ora_map* m) { return m->err.c_str(); }

static std::string validate_frame(const ora_config& c, const ora_frame* f) {
  if (!f) return "null frame";
  if (f->height <= 0 || f->width <= 0) return "bad image dims";
  if (!f->depth) return "null depth";
  if (f->num_masks < 0) return "negative num_masks";
  if (f->num_masks > 0 && !f->masks) return "null masks";
  if (f->patch_h < 1 || f->patch_h > f->height || f->patch_w < 1 || f->patch_w > f->width)
    return "bad patch grid";
  if (c.track_dim > 0 && !f->track_feats) return "track_dim > 0 requires track_feats";
  if (!(f->fx != 0.0f && f->fy != 0.0f) || !std::isfinite(f->fx) || !std::isfinite(f->fy))
    return "bad intrinsics";
  if (!ora_pose_rigid(f->pose)) return "non-rigid pose";
  return "";
}

static void aabb_of(const std::set<Key>& V, int32_t out[6]) {
  out[0] = out[1] = out[2] = INT32_MAX;
  out[3] = out[4] = out[5] = INT32_MIN;
  for (const Key& k : V)
    for (int i = 0; i < 3; ++i) {
      out[i] = std::min(out[i], k[i]);
      out[3 + i] = std::max(out[3 + i], k[i]);
    }
}

static void add_accept(Inst& I, double q, const std::vector<double>& e) {
  if (q < 0.0) return;  // observation without embedding
  I.accept.push_back({q, e});
  double qmax = -1.0;
  for (const Obs& o : I.accept) qmax = std::max(qmax, o.q);
  std::vector<Obs> kept;
  for (Obs& o : I.accept)
    if (o.q >= qmax * (1.0 - 1e-4)) kept.push_back(std::move(o));
  I.accept.swap(kept);
}

extern "C" int32_t ora_integrate(ora_map* m, const ora_frame* f, ora_report* rep) {
  const ora_config& c = m->cfg;
  /* O0 validate (A0): on failure the state is untouched */
  std::string verr = validate_frame(c, f);
  if (!verr.empty()) {
    m->err = verr;
    return ORA_INVALID;
  }
  m->err.clear();
  const int32_t H = f->height, W = f->width, S = f->num_masks;
  const int32_t Hp = f->patch_h, Wp = f->patch_w;
  const int64_t P = (int64_t)Hp * Wp, HW = (int64_t)H * W;
  const int32_t Df = c.feat_dim, Dt = c.track_dim;
  const bool semantic = f->patch_feats != nullptr;
  ora_report R{};
  std::vector<Det> det(S);

  /* O1 mask stats and filter (R8) */
  for (int32_t s = 0; s < S; ++s) {
    Det& d = det[s];
    int32_t umin = INT32_MAX, vmin = INT32_MAX, umax = -1, vmax = -1;
    const uint8_t* M = f->masks + (int64_t)s * HW;
    for (int32_t v = 0; v < H; ++v)
      for (int32_t u = 0; u < W; ++u)
        if (M[(int64_t)v * W + u]) {
          d.area++;
          umin = std::min(umin, u); umax = std::max(umax, u);
          vmin = std::min(vmin, v); vmax = std::max(vmax, v);
        }
    if (d.area > 0) {
      d.bbox[0] = umin; d.bbox[1] = vmin; d.bbox[2] = umax; d.bbox[3] = vmax;
    }
    const float conf = f->mask_conf ? f->mask_conf[s] : 1.0f;
    if (d.area == 0) { d.status = ORA_DROP_AREA; continue; }
    if (conf < c.mask_min_conf) { d.status = ORA_DROP_CONF; continue; }
    const int64_t bw = umax - umin + 1, bh = vmax - vmin + 1;
    const int64_t lo = std::min(bw, bh), hi = std::max(bw, bh);
    // aspect = hi/lo > max_aspect, decided exactly in fp64 (hi, lo < 2^24)
    if ((double)hi > (double)c.mask_max_aspect * (double)lo) { d.status = ORA_DROP_ASPECT; continue; }
    if (d.area < c.mask_min_area) { d.status = ORA_DROP_AREA; continue; }
  }

  /* O2 points and keys (R5, R6) */
  std::vector<std::array<float, 3>> pw(HW);
  std::vector<uint8_t> dvalid(HW, 0), kvalid(HW, 0);
  std::vector<Key> key(HW);
  for (int32_t v = 0; v < H; ++v)
    for (int32_t u = 0; u < W; ++u) {
      const int64_t i = (int64_t)v * W + u;
      if (!ora_pixel_world(&c, f, u, v, pw[i].data())) continue;
      dvalid[i] = 1;
      if (ora_point_key(pw[i].data(), c.voxel_size, key[i].data())) kvalid[i] = 1;
      else R.key_out_of_range++;
    }
  const double cam[3] = {(double)f->pose[3], (double)f->pose[7], (double)f->pose[11]};

  /* O4 pixel normals (R21): n = (P(u+1,v)-P(u-1,v)) x (P(u,v+1)-P(u,v-1)), 4 valid
   * in-image neighbours, oriented so n.(cam - P) >= 0; zero vector = no normal. */
  auto pixel_normal = [&](int32_t u, int32_t v, double n[3]) -> bool {
    if (u < 1 || u + 1 >= W || v < 1 || v + 1 >= H) return false;
    const int64_t i = (int64_t)v * W + u;
    const int64_t iL = i - 1, iR = i + 1, iU = i - W, iD = i + W;
    if (!dvalid[iL] || !dvalid[iR] || !dvalid[iU] || !dvalid[iD]) return false;
    double a[3], b[3];
    for (int k = 0; k < 3; ++k) {
      a[k] = (double)pw[iR][k] - (double)pw[iL][k];
      b[k] = (double)pw[iD][k] - (double)pw[iU][k];
    }
    n[0] = a[1] * b[2] - a[2] * b[1];
    n[1] = a[2] * b[0] - a[0] * b[2];
    n[2] = a[0] * b[1] - a[1] * b[0];
    if (n[0] == 0.0 && n[1] == 0.0 && n[2] == 0.0) return false;
    const double o = n[0] * (cam[0] - pw[i][0]) + n[1] * (cam[1] - pw[i][1]) + n[2] * (cam[2] - pw[i][2]);
    if (o < 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
    return true;
  };

  /* O3 detection voxel sets V_s, with O4 normal sums per (s, k).  With DBSCAN on (R42): only
   * the pixels whose world points form the segment's largest DBSCAN cluster (by point count; ties:
   * the first cluster created) contribute; a segment left without points is dropped ("nodepth"). */
  for (int32_t s = 0; s < S; ++s) {
    Det& d = det[s];
    if (d.status != ORA_KEPT) continue;
    const uint8_t* M = f->masks + (int64_t)s * HW;
    std::vector<uint8_t> keep;   // DBSCAN: pixels of the kept cluster
    if (c.dbscan_eps > 0.0f) {
      std::vector<int64_t> pix;
      std::vector<float> P3;
      for (int64_t i = 0; i < HW; ++i)
        if (M[i] && kvalid[i]) {
          pix.push_back(i);
          P3.insert(P3.end(), pw[i].begin(), pw[i].end());
        }
      std::vector<int32_t> lab(pix.size());
      const int32_t nc = ora_dbscan((int64_t)pix.size(), P3.data(), c.dbscan_eps, c.dbscan_min_pts, lab.data());
      std::vector<int64_t> size(nc, 0);
      for (int32_t l : lab)
        if (l >= 0) size[l]++;
      int32_t best = -1;
      for (int32_t k = 0; k < nc; ++k)
        if (best < 0 || size[k] > size[best]) best = k;
      keep.assign(HW, 0);
      for (size_t q = 0; q < pix.size(); ++q)
        if (best >= 0 && lab[q] == best) keep[pix[q]] = 1;
    }
    for (int32_t v = 0; v < H; ++v)
      for (int32_t u = 0; u < W; ++u) {
        const int64_t i = (int64_t)v * W + u;
        if (!M[i] || !kvalid[i]) continue;
        if (!keep.empty() && !keep[i]) continue;
        d.V.insert(key[i]);
        if (semantic) {
          double n[3];
          if (pixel_normal(u, v, n)) {
            auto& acc = d.nsum[key[i]];
            acc[0] += n[0]; acc[1] += n[1]; acc[2] += n[2];
            d.nnorm[key[i]]++;
          }
        }
      }
    if (d.V.empty()) d.status = ORA_DROP_NODEPTH;
  }

  /* O5 patch mapping (R17): p(v,u) = (floor(v Hp / H), floor(u Wp / W)) */
  std::vector<int64_t> npix(P, 0);
  std::vector<int64_t> pidx(HW);
  for (int32_t v = 0; v < H; ++v)
    for (int32_t u = 0; u < W; ++u) {
      const int64_t pi = ((int64_t)v * Hp / H) * Wp + ((int64_t)u * Wp / W);
      pidx[(int64_t)v * W + u] = pi;
      npix[pi]++;
    }
  std::vector<std::vector<int64_t>> cnt(S);  // cnt_sp, counted regardless of depth
  for (int32_t s = 0; s < S; ++s) {
    if (det[s].status != ORA_KEPT) continue;
    cnt[s].assign(P, 0);
    const uint8_t* M = f->masks + (int64_t)s * HW;
    for (int64_t i = 0; i < HW; ++i)
      if (M[i]) cnt[s][pidx[i]]++;
  }

  /* O6 distinctiveness and O7 feature + quality (only with patch features) */
  if (semantic) {
    std::vector<double> D(P);
    ora_distinctiveness(P, Df, f->patch_feats, (double)c.eps_distinct, D.data());
    for (int32_t s = 0; s < S; ++s) {
      Det& d = det[s];
      if (d.status != ORA_KEPT) continue;
      d.e.assign(Df, 0.0);
      double dbar = 0.0;
      if (ora_pool(P, Df, cnt[s].data(), npix.data(), D.data(), f->patch_feats,
                   (double)c.cover_min, d.e.data(), &dbar)) {
        d.status = ORA_DROP_NOFEAT;
        continue;
      }
      const double s_size = ora_s_size(d.area, H, W, (double)c.lambda_size);
      // S_angle (Eq.3, R21): voxels with a non-zero normal sum; ray from camera centre to
      // voxel centre (k + 0.5) r
      std::vector<double> nn, rr;
      const double r = (double)c.voxel_size;
      for (const Key& k : d.V) {
        auto it = d.nsum.find(k);
        if (it == d.nsum.end()) continue;
        const auto& ns = it->second;
        const double l = std::sqrt(ns[0] * ns[0] + ns[1] * ns[1] + ns[2] * ns[2]);
        if (l == 0.0) continue;
        double ray[3];
        for (int a = 0; a < 3; ++a) ray[a] = ((double)k[a] + 0.5) * r - cam[a];
        const double rl = std::sqrt(ray[0] * ray[0] + ray[1] * ray[1] + ray[2] * ray[2]);
        if (rl == 0.0) continue;
        for (int a = 0; a < 3; ++a) {
          nn.push_back(ns[a] / l);
          rr.push_back(ray[a] / rl);
        }
      }
      const double s_angle = ora_s_angle((int64_t)(nn.size() / 3), nn.data(), rr.data());
      const double s_sem = ora_s_sem(Df, d.e.data(), f->global_embed);
      const double s_dist = ora_s_dist(dbar);
      d.f[0] = s_size; d.f[1] = s_angle; d.f[2] = s_sem; d.f[3] = s_dist;
      d.f[4] = ora_quality(s_size, s_angle, s_sem, s_dist);
      d.f[5] = dbar;
    }
  } else {
    for (int32_t s = 0; s < S; ++s) det[s].e.assign(Df, 0.0);
  }

  /* O8 tracking (R15): u_s = sum_p cnt_sp g_p in fp64; t_s = u_s / sqrt(dot_pin(u_s,u_s)) */
  if (Dt > 0) {
    for (int32_t s = 0; s < S; ++s) {
      Det& d = det[s];
      if (d.status != ORA_KEPT) continue;
      d.u.assign(Dt, 0.0);
      d.t.assign(Dt, 0.0);
      for (int64_t p = 0; p < P; ++p) {
        if (cnt[s][p] == 0) continue;
        for (int32_t k = 0; k < Dt; ++k)
          d.u[k] += (double)cnt[s][p] * bf16_to_double(f->track_feats[p * Dt + k]);
      }
      const double nn = ora_dot_pin(Dt, d.u.data(), d.u.data());
      if (nn > 0.0) {
        const double n = std::sqrt(nn);
        for (int32_t k = 0; k < Dt; ++k) d.t[k] = d.u[k] / n;
        d.t_ok = true;
      }
    }
  }

  /* O9 overlaps c_sj = |V_s ∩ V_j| against the frame-start map (inverted index; the
   * self-check recomputes every (s,j) by std::set_intersection) */
  std::map<std::pair<int32_t, Id>, int64_t> C;
  for (int32_t s = 0; s < S; ++s) {
    if (det[s].status != ORA_KEPT) continue;
    for (const Key& k : det[s].V) {
      auto it = m->mem.find(k);
      if (it == m->mem.end()) continue;
      for (Id j : it->second) C[{s, j}]++;
    }
  }
  if (m->selfcheck) {
    std::map<std::pair<int32_t, Id>, int64_t> Cb;
    for (int32_t s = 0; s < S; ++s) {
      if (det[s].status != ORA_KEPT) continue;
      for (const auto& kv : m->inst) {
        std::vector<Key> out;
        std::set_intersection(det[s].V.begin(), det[s].V.end(), kv.second.V.begin(),
                              kv.second.V.end(), std::back_inserter(out));
        if (!out.empty()) Cb[{s, kv.first}] = (int64_t)out.size();
      }
    }
    if (Cb != C) {
      m->err = "selfcheck: inverted-index overlap counts != set_intersection";
      return ORA_SELFCHECK_FAILED;
    }
  }

  /* O10 edges (R10 exact fp64 threshold, R15 pinned gate) */
  std::set<std::pair<int32_t, Id>> E;
  for (const auto& kv : C) {
    const int32_t s = kv.first.first;
    const Id j = kv.first.second;
    const int64_t cij = kv.second;
    const Inst& I = m->inst.at(j);
    const int64_t mn = std::min((int64_t)det[s].V.size(), (int64_t)I.V.size());
    if (!(cij >= 1 && (double)cij >= (double)c.tau_geo * (double)mn)) continue;
    if (Dt > 0) {
      double cosv = -2.0;
      const double TT = ora_dot_pin(Dt, I.T.data(), I.T.data());
      if (det[s].t_ok && TT > 0.0) cosv = ora_dot_pin(Dt, det[s].t.data(), I.T.data()) / std::sqrt(TT);
      if (!(cosv >= (double)c.tau_vis)) continue;
    }
    E.insert({s, j});
  }
  R.edges = (int64_t)E.size();

  /* O11 components: BFS over kept detections ∪ instances with edges E.
   * node encoding: detection s -> (0, s), instance j -> (1, j) */
  using Node = std::pair<int, int64_t>;
  std::map<Node, std::vector<Node>> adj;
  for (const auto& e : E) {
    adj[{0, e.first}].push_back({1, e.second});
    adj[{1, e.second}].push_back({0, e.first});
  }
  std::map<Node, int64_t> comp;
  int64_t ncomp = 0;
  for (const auto& kv : adj) {
    if (comp.count(kv.first)) continue;
    std::deque<Node> q{kv.first};
    comp[kv.first] = ncomp;
    while (!q.empty()) {
      Node x = q.front();
      q.pop_front();
      for (const Node& y : adj[x])
        if (!comp.count(y)) { comp[y] = ncomp; q.push_back(y); }
    }
    ncomp++;
  }
  if (m->selfcheck) {  // union-find must give the same partition as BFS
    std::map<Node, Node> par;
    std::function<Node(Node)> find = [&](Node x) -> Node {
      auto it = par.find(x);
      if (it == par.end()) { par[x] = x; return x; }
      if (it->second == x) return x;
      Node r = find(it->second);
      par[x] = r;
      return r;
    };
    for (const auto& e : E) {
      Node a = find({0, e.first}), b = find({1, e.second});
      if (a != b) par[std::max(a, b)] = std::min(a, b);
    }
    for (const auto& x : comp)
      for (const auto& y : comp)
        if ((x.second == y.second) != (find(x.first) == find(y.first))) {
          m->err = "selfcheck: union-find partition != BFS partition";
          return ORA_SELFCHECK_FAILED;
        }
  }

  /* O12 apply */
  int64_t live_before = 0;
  for (const auto& kv : m->inst) live_before += (int64_t)kv.second.V.size();
  std::map<Id, Id> merged_into;   // O12's erased ids -> their component root (refinement, R43)
  std::vector<std::vector<Id>> cJ(ncomp);
  std::vector<std::vector<int32_t>> cS(ncomp);
  for (const auto& kv : comp) {
    if (kv.first.first == 0) cS[kv.second].push_back((int32_t)kv.first.second);
    else cJ[kv.second].push_back(kv.first.second);
  }
  for (int64_t ci = 0; ci < ncomp; ++ci) {
    std::vector<Id>& J = cJ[ci];
    std::vector<int32_t>& Sd = cS[ci];
    std::sort(J.begin(), J.end());
    std::sort(Sd.begin(), Sd.end());
    const Id root = J.front();
    Inst& Rt = m->inst.at(root);
    // voxel union
    for (size_t a = 1; a < J.size(); ++a) {
      const Inst& Ij = m->inst.at(J[a]);
      R.relabeled += (int64_t)Ij.V.size();
      Rt.V.insert(Ij.V.begin(), Ij.V.end());
    }
    for (int32_t s : Sd) Rt.V.insert(det[s].V.begin(), det[s].V.end());
    // counts
    for (size_t a = 1; a < J.size(); ++a) Rt.obs += m->inst.at(J[a]).obs;
    Rt.obs += (int32_t)Sd.size();
    Rt.last_seen = f->frame_id;
    // T: ((T_root + T_j1) + T_j2 ...) + t_s1 ...  elementwise fp64, in exactly this order
    if (Dt > 0) {
      for (size_t a = 1; a < J.size(); ++a) {
        const Inst& Ij = m->inst.at(J[a]);
        for (int32_t k = 0; k < Dt; ++k) Rt.T[k] = Rt.T[k] + Ij.T[k];
      }
      for (int32_t s : Sd)
        for (int32_t k = 0; k < Dt; ++k) Rt.T[k] = Rt.T[k] + det[s].t[k];
    }
    // (e, Q): root's, then each j in J, then each s in Sd: replace iff Q_cand > Q (strict)
    for (size_t a = 1; a < J.size(); ++a) {
      Inst& Ij = m->inst.at(J[a]);
      if (Ij.Q > Rt.Q) { Rt.Q = Ij.Q; Rt.e = Ij.e; }
      for (Obs& o : Ij.accept) add_accept(Rt, o.q, o.e);
    }
    for (int32_t s : Sd) {
      const double qs = semantic ? det[s].f[4] : -1.0;
      if (qs > Rt.Q) { Rt.Q = qs; Rt.e = det[s].e; }
      if (semantic) add_accept(Rt, qs, det[s].e);
      det[s].target = root;
    }
    // erase J \ {root}; membership relation rewritten to root
    for (size_t a = 1; a < J.size(); ++a) {
      const Inst& Ij = m->inst.at(J[a]);
      for (const Key& k : Ij.V) {
        auto& ids = m->mem[k];
        ids.erase(J[a]);
        ids.insert(root);
      }
      m->inst.erase(J[a]);
      merged_into[J[a]] = root;
      R.merged_away++;
    }
    for (int32_t s : Sd)
      for (const Key& k : det[s].V) m->mem[k].insert(root);
  }
  // isolated kept detections -> new instances, ascending s (R13)
  for (int32_t s = 0; s < S; ++s) {
    Det& d = det[s];
    if (d.status != ORA_KEPT) continue;
    if (comp.count({0, s})) continue;
    const Id id = m->next_id++;
    Inst I;
    I.V = d.V;
    I.obs = 1;
    I.last_seen = f->frame_id;
    I.Q = semantic ? d.f[4] : -1.0;
    I.e = d.e;
    I.T = Dt > 0 ? d.t : std::vector<double>();
    if (semantic) add_accept(I, I.Q, d.e);
    for (const Key& k : d.V) m->mem[k].insert(id);
    m->inst.emplace(id, std::move(I));
    d.target = id;
    R.created++;
  }

  /* R43 (refine_active; S:327 step (3) "within the active set, merge existing instance pairs meeting
   * the same (tau_geo, tau_vis) test, keeping the lower id and the higher-Q semantic feature; repeat
   * pairwise merging until no pair qualifies"; "merged ... among all candidates").  Active set =
   * the instances the frame's detections overlapped (the C triples' j, taken to their O12 survivor)
   * and the frame's targets (survivors and new ids).  Rounds of R35's snapshot union-find over the
   * active pairs (R36's test on c_ij = |V_i ∩ V_j|, R37's merge), the active set taken to the
   * survivors after each round, until no active pair qualifies. */
  if (c.refine_active) {
    std::set<Id> A;
    for (const auto& kv : C) {
      Id j = kv.first.second;
      auto it = merged_into.find(j);
      A.insert(it == merged_into.end() ? j : it->second);
    }
    for (int32_t s = 0; s < S; ++s)
      if (det[s].status == ORA_KEPT && det[s].target >= 0) A.insert(det[s].target);
    while (true) {
      std::map<Id, std::vector<Id>> adj;
      int64_t nedge = 0;
      for (auto ia = A.begin(); ia != A.end(); ++ia)
        for (auto ib = std::next(ia); ib != A.end(); ++ib) {
          const Inst& I = m->inst.at(*ia);
          const Inst& J2 = m->inst.at(*ib);
          std::vector<Key> out;
          std::set_intersection(I.V.begin(), I.V.end(), J2.V.begin(), J2.V.end(), std::back_inserter(out));
          const int64_t cij = (int64_t)out.size();
          const int64_t mn = std::min((int64_t)I.V.size(), (int64_t)J2.V.size());
          if (!(cij >= 1 && (double)cij >= (double)c.tau_geo * (double)mn)) continue;
          if (Dt > 0) {
            const double aa = ora_dot_pin(Dt, I.T.data(), I.T.data());
            const double bb = ora_dot_pin(Dt, J2.T.data(), J2.T.data());
            double cosv = -2.0;
            if (aa > 0.0 && bb > 0.0) cosv = ora_dot_pin(Dt, I.T.data(), J2.T.data()) / std::sqrt(aa) / std::sqrt(bb);
            if (!(cosv >= (double)c.tau_vis)) continue;
          }
          adj[*ia].push_back(*ib);
          adj[*ib].push_back(*ia);
          nedge++;
        }
      if (nedge == 0) break;
      R.refine_rounds++;
      std::set<Id> seen;
      std::map<Id, Id> root_of;
      for (const auto& kv : adj) {
        if (seen.count(kv.first)) continue;
        std::vector<Id> comp;
        std::deque<Id> q{kv.first};
        seen.insert(kv.first);
        while (!q.empty()) {
          const Id x = q.front();
          q.pop_front();
          comp.push_back(x);
          for (Id y : adj[x])
            if (!seen.count(y)) { seen.insert(y); q.push_back(y); }
        }
        std::sort(comp.begin(), comp.end());
        const Id root = comp.front();
        Inst& Rt = m->inst.at(root);
        for (size_t a = 1; a < comp.size(); ++a) {
          Inst& Ij = m->inst.at(comp[a]);
          R.relabeled += (int64_t)Ij.V.size();
          Rt.V.insert(Ij.V.begin(), Ij.V.end());
          Rt.obs += Ij.obs;
          Rt.last_seen = std::max(Rt.last_seen, Ij.last_seen);
          for (int32_t k = 0; k < Dt; ++k) Rt.T[k] = Rt.T[k] + Ij.T[k];
          if (Ij.Q > Rt.Q) { Rt.Q = Ij.Q; Rt.e = Ij.e; }
          for (Obs& o : Ij.accept) add_accept(Rt, o.q, o.e);
          for (const Key& k : Ij.V) {
            auto& ids = m->mem[k];
            ids.erase(comp[a]);
            ids.insert(root);
          }
          m->inst.erase(comp[a]);
          root_of[comp[a]] = root;
          R.merged_away++;
          R.refine_merged++;
        }
        for (int32_t s = 0; s < S; ++s)
          if (det[s].target >= 0 && root_of.count(det[s].target)) det[s].target = root;
      }
      std::set<Id> A2;
      for (Id a : A) A2.insert(root_of.count(a) ? root_of[a] : a);
      A.swap(A2);
    }
  }

  /* O13 report */
  for (int32_t s = 0; s < S; ++s) {
    switch (det[s].status) {
      case ORA_KEPT: R.kept++; R.unique_pairs += (int64_t)det[s].V.size(); break;
      case ORA_DROP_AREA: R.drop_area++; break;
      case ORA_DROP_CONF: R.drop_conf++; break;
      case ORA_DROP_ASPECT: R.drop_aspect++; break;
      case ORA_DROP_NODEPTH: R.drop_nodepth++; break;
      case ORA_DROP_NOFEAT: R.drop_nofeat++; break;
    }
  }
  int64_t live_after = 0;
  for (const auto& kv : m->inst) live_after += (int64_t)kv.second.V.size();
  R.live_instances = (int64_t)m->inst.size();
  R.live_memberships = live_after;
  R.new_memberships = live_after - live_before;

  if (m->selfcheck) {  // C.4 map invariants
    int64_t rel = 0;
    for (const auto& kv : m->mem) {
      for (Id j : kv.second) {
        auto it = m->inst.find(j);
        if (it == m->inst.end() || !it->second.V.count(kv.first)) {
          m->err = "selfcheck: membership relation and instance voxel sets disagree";
          return ORA_SELFCHECK_FAILED;
        }
      }
      rel += (int64_t)kv.second.size();
    }
    if (rel != live_after) {
      m->err = "selfcheck: live memberships != sum |V_j|";
      return ORA_SELFCHECK_FAILED;
    }
  }
  m->last = std::move(det);
  m->last_c = std::move(C);
  m->last_edges = std::move(E);
  if (rep) *rep = R;
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* finalize (NEXT f1): P:100 [§III-B] "a final, lightweight post-processing step iterates   */
/* over the map to merge remaining orphaned candidates and filter out residual noisy        */
/* instances, such as segments containing fewer than a minimum threshold of voxels";        */
/* S:333-337 "all instance pairs meeting (tau_geo, tau_vis) merged to fixpoint ...; then     */
/* every instance with |voxels| < min_voxels removed".  Readings:              */
/*  R35 fixpoint = rounds of the snapshot union-find of R12 over INSTANCE pairs: each round */
/*      tests every pair against the round-start map, merges each component into its min  */
/*      id, and the rounds repeat until no pair qualifies;                                  */
/*  R36 pair test = R10's c >= 1 and c >= tau_geo min(|V_i|, |V_j|) exactly in fp64, with  */
/*      c = |V_i ∩ V_j|, and (Dt > 0) the gate (dot_pin(T_i,T_j) / sqrt(dot_pin(T_i,T_i)))  */
/*      / sqrt(dot_pin(T_j,T_j)) >= tau_vis for i < j, a zero norm giving -2 (R15 pinned);  */
/*  R37 merge = O12 without detections: V union, obs summed, last_seen = max, T summed in   */
/*      ascending id order, (e, Q) replaced in ascending id order iff Q_j > Q (strict);     */
/*  R38 the filter runs once, after the fixpoint; removed instances lose their memberships. */
/* ------------------------------------------------------------------------------------ */
extern "C" int32_t ora_finalize(ora_map* m, float tau_geo, float tau_vis, int64_t min_voxels,
                                ora_final_report* rep) {
  ora_final_report R{};
  const int32_t Dt = m->cfg.track_dim;
  while (true) {
    /* pair counts c_ij = |V_i ∩ V_j| from the membership relation (every key's id set) */
    std::map<std::pair<Id, Id>, int64_t> C;
    for (const auto& kv : m->mem) {
      const std::vector<Id> ids(kv.second.begin(), kv.second.end());  // ascending
      for (size_t a = 0; a < ids.size(); ++a)
        for (size_t b = a + 1; b < ids.size(); ++b) C[{ids[a], ids[b]}]++;
    }
    if (m->selfcheck) {  // brute force: std::set_intersection over every pair of instances
      for (auto i = m->inst.begin(); i != m->inst.end(); ++i)
        for (auto j = std::next(i); j != m->inst.end(); ++j) {
          std::vector<Key> out;
          std::set_intersection(i->second.V.begin(), i->second.V.end(), j->second.V.begin(),
                                j->second.V.end(), std::back_inserter(out));
          auto it = C.find({i->first, j->first});
          if ((int64_t)out.size() != (it == C.end() ? 0 : it->second)) {
            m->err = "selfcheck: finalize pair counts != set_intersection";
            return ORA_SELFCHECK_FAILED;
          }
        }
    }
    /* R36 qualifying pairs */
    std::map<Id, std::vector<Id>> adj;
    int64_t nedge = 0;
    for (const auto& kv : C) {
      const Id i = kv.first.first, j = kv.first.second;
      const Inst& A = m->inst.at(i);
      const Inst& B = m->inst.at(j);
      const int64_t c = kv.second;
      const int64_t mn = std::min((int64_t)A.V.size(), (int64_t)B.V.size());
      if (!(c >= 1 && (double)c >= (double)tau_geo * (double)mn)) continue;
      if (Dt > 0) {
        const double aa = ora_dot_pin(Dt, A.T.data(), A.T.data());
        const double bb = ora_dot_pin(Dt, B.T.data(), B.T.data());
        double cosv = -2.0;
        if (aa > 0.0 && bb > 0.0) cosv = ora_dot_pin(Dt, A.T.data(), B.T.data()) / std::sqrt(aa) / std::sqrt(bb);
        if (!(cosv >= (double)tau_vis)) continue;
      }
      adj[i].push_back(j);
      adj[j].push_back(i);
      nedge++;
    }
    if (nedge == 0) break;
    R.rounds++;
    R.edges += nedge;
    /* components (BFS), each merged into its min id (R37) */
    std::set<Id> seen;
    std::vector<std::vector<Id>> comps;
    for (const auto& kv : adj) {
      if (seen.count(kv.first)) continue;
      std::vector<Id> comp;
      std::deque<Id> q{kv.first};
      seen.insert(kv.first);
      while (!q.empty()) {
        const Id x = q.front();
        q.pop_front();
        comp.push_back(x);
        for (Id y : adj[x])
          if (!seen.count(y)) { seen.insert(y); q.push_back(y); }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(comp);
    }
    for (const auto& J : comps) {
      const Id root = J.front();
      Inst& Rt = m->inst.at(root);
      for (size_t a = 1; a < J.size(); ++a) {
        Inst& Ij = m->inst.at(J[a]);
        R.relabeled += (int64_t)Ij.V.size();
        Rt.V.insert(Ij.V.begin(), Ij.V.end());
        Rt.obs += Ij.obs;
        Rt.last_seen = std::max(Rt.last_seen, Ij.last_seen);
        for (int32_t k = 0; k < Dt; ++k) Rt.T[k] = Rt.T[k] + Ij.T[k];
        if (Ij.Q > Rt.Q) { Rt.Q = Ij.Q; Rt.e = Ij.e; }
        for (Obs& o : Ij.accept) add_accept(Rt, o.q, o.e);
        for (const Key& k : Ij.V) {
          auto& ids = m->mem[k];
          ids.erase(J[a]);
          ids.insert(root);
        }
        m->inst.erase(J[a]);
        R.merged_away++;
      }
    }
  }
  /* R38 the minimum-size filter */
  std::vector<Id> drop;
  for (const auto& kv : m->inst)
    if ((int64_t)kv.second.V.size() < min_voxels) drop.push_back(kv.first);
  for (Id id : drop) {
    for (const Key& k : m->inst.at(id).V) {
      auto it = m->mem.find(k);
      it->second.erase(id);
      if (it->second.empty()) m->mem.erase(it);
    }
    m->inst.erase(id);
    R.removed++;
  }
  R.live_instances = (int64_t)m->inst.size();
  for (const auto& kv : m->inst) R.live_memberships += (int64_t)kv.second.V.size();
  if (rep) *rep = R;
  return ORA_OK;
}

/* ------------------------------------------------------------------------------------ */
/* export                                                                                */
/* ------------------------------------------------------------------------------------ */

extern "C" int64_t ora_num_instances(const ora_map* m) { return (int64_t)m->inst.size(); }
extern "C" int64_t ora_next_id(const ora_map* m) { return m->next_id; }

extern "C" int64_t ora_get_instances(const ora_map* m, int64_t* id, int64_t* vcount, int32_t* obs,
                                     int64_t* last_seen, double* q, int32_t* aabb6, double* e,
                                     double* T, int64_t cap) {
  const int32_t Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  int64_t n = 0;
  for (const auto& kv : m->inst) {  // std::map: ascending id
    if (n >= cap) break;
    const Inst& I = kv.second;
    if (id) id[n] = kv.first;
    if (vcount) vcount[n] = (int64_t)I.V.size();
    if (obs) obs[n] = I.obs;
    if (last_seen) last_seen[n] = I.last_seen;
    if (q) q[n] = I.Q;
    if (aabb6) aabb_of(I.V, aabb6 + 6 * n);
    if (e)
      for (int32_t d = 0; d < Df; ++d) e[n * Df + d] = I.Q >= 0.0 ? I.e[d] : 0.0;
    if (T)
      for (int32_t d = 0; d < Dt; ++d) T[n * Dt + d] = I.T[d];
    n++;
  }
  return n;
}

extern "C" int64_t ora_num_memberships(const ora_map* m) {
  int64_t n = 0;
  for (const auto& kv : m->mem) n += (int64_t)kv.second.size();
  return n;
}

extern "C" int64_t ora_get_memberships(const ora_map* m, uint64_t* keys, int64_t* ids, int64_t cap) {
  int64_t n = 0;
  for (const auto& kv : m->mem)
    for (Id j : kv.second) {
      if (n >= cap) return n;
      keys[n] = pack(kv.first);
      ids[n] = j;
      n++;
    }
  return n;
}

extern "C" int64_t ora_get_accept(const ora_map* m, int64_t id, double* q, double* e, int64_t cap) {
  auto it = m->inst.find(id);
  if (it == m->inst.end()) return -1;
  const int32_t Df = m->cfg.feat_dim;
  int64_t n = 0;
  for (const Obs& o : it->second.accept) {
    if (n >= cap) break;
    if (q) q[n] = o.q;
    if (e)
      for (int32_t d = 0; d < Df; ++d) e[n * Df + d] = o.e[d];
    n++;
  }
  return (int64_t)it->second.accept.size();
}

extern "C" int32_t ora_last_num_masks(const ora_map* m) { return (int32_t)m->last.size(); }

extern "C" void ora_last_masks(const ora_map* m, int32_t* status, int64_t* area, int32_t* bbox4,
                               int64_t* vs, int64_t* target) {
  for (size_t s = 0; s < m->last.size(); ++s) {
    const Det& d = m->last[s];
    if (status) status[s] = d.status;
    if (area) area[s] = d.area;
    if (bbox4)
      for (int k = 0; k < 4; ++k) bbox4[4 * s + k] = d.bbox[k];
    if (vs) vs[s] = (int64_t)d.V.size();
    if (target) target[s] = d.target;
  }
}

extern "C" int64_t ora_last_pairs(const ora_map* m, int32_t* s, uint64_t* keys, int64_t cap) {
  int64_t n = 0;
  for (size_t i = 0; i < m->last.size(); ++i) {
    const Det& d = m->last[i];
    if (d.status != ORA_KEPT) continue;
    for (const Key& k : d.V) {
      if (n < cap && s) { s[n] = (int32_t)i; keys[n] = pack(k); }
      n++;
    }
  }
  return n;
}

extern "C" int64_t ora_last_triples(const ora_map* m, int32_t* s, int64_t* j, int64_t* c,
                                    int32_t* edge, int64_t cap) {
  int64_t n = 0;
  for (const auto& kv : m->last_c) {
    if (n < cap && s) {
      s[n] = kv.first.first;
      j[n] = kv.first.second;
      c[n] = kv.second;
      edge[n] = m->last_edges.count(kv.first) ? 1 : 0;
    }
    n++;
  }
  return n;
}

extern "C" void ora_last_quality(const ora_map* m, double* f6, double* e, double* u, double* t) {
  const int32_t Df = m->cfg.feat_dim, Dt = m->cfg.track_dim;
  for (size_t s = 0; s < m->last.size(); ++s) {
    const Det& d = m->last[s];
    if (f6)
      for (int k = 0; k < 6; ++k) f6[6 * s + k] = d.f[k];
    if (e)
      for (int32_t k = 0; k < Df; ++k) e[s * Df + k] = (int32_t)d.e.size() == Df ? d.e[k] : 0.0;
    if (u)
      for (int32_t k = 0; k < Dt; ++k) u[s * Dt + k] = (int32_t)d.u.size() == Dt ? d.u[k] : 0.0;
    if (t)
      for (int32_t k = 0; k < Dt; ++k) t[s * Dt + k] = (int32_t)d.t.size() == Dt ? d.t[k] : 0.0;
  }
}

/* Q1: score_j = e_j . q/|q| over live instances with an embedding;
 * full sort by descending score, ties by ascending id. */
extern "C" int64_t ora_query(const ora_map* m, const float* q, int32_t k, int64_t* ids,
                             double* scores) {
  const int32_t Df = m->cfg.feat_dim;
  double qq = 0.0;
  for (int32_t d = 0; d < Df; ++d) qq += (double)q[d] * (double)q[d];
  const double qn = std::sqrt(qq);
  std::vector<std::pair<double, Id>> all;
  for (const auto& kv : m->inst) {
    if (kv.second.Q < 0.0) continue;
    double s = 0.0;
    for (int32_t d = 0; d < Df; ++d) s += kv.second.e[d] * ((double)q[d] / qn);
    all.push_back({s, kv.first});
  }
  std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) {
    if (a.first != b.first) return a.first > b.first;
    return a.second < b.second;
  });
  int64_t n = std::min<int64_t>(k, (int64_t)all.size());
  for (int64_t i = 0; i < n; ++i) {
    ids[i] = all[i].second;
    scores[i] = all[i].first;
  }
  return n;
}

/* ------------------------------------------------------------------------------------ */
/* batched open-vocabulary retrieval (NEXT f4): P:195 [§IV-A] "the correct ground-truth     */
/* semantic class appearing within the top-k cosine-similarity predictions"      */
/* classify_topk: "indices of the k largest cosines against table rows, descending, ties by */
/* ascending index", for every live instance with an embedding (ascending id).  R39: the     */
/* cosine is e_j . t_c / |t_c| in fp64 (e_j is unit, Eq. of S:391's rank_instances).         */
/* ------------------------------------------------------------------------------------ */
extern "C" int64_t ora_classify(const ora_map* m, const float* table, int32_t C, int32_t k, int64_t* ids,
                                int32_t* classes, double* scores, int64_t cap) {
  const int32_t Df = m->cfg.feat_dim;
  std::vector<double> tn(C);
  for (int32_t c = 0; c < C; ++c) {
    double t = 0.0;
    for (int32_t d = 0; d < Df; ++d) t += (double)table[(int64_t)c * Df + d] * (double)table[(int64_t)c * Df + d];
    tn[c] = std::sqrt(t);
  }
  const int32_t kk = std::min(k, C);
  int64_t n = 0;
  for (const auto& kv : m->inst) {
    if (kv.second.Q < 0.0) continue;
    if (n < cap && ids) {
      std::vector<std::pair<double, int32_t>> all(C);
      for (int32_t c = 0; c < C; ++c) {
        double s = 0.0;
        for (int32_t d = 0; d < Df; ++d) s += kv.second.e[d] * (double)table[(int64_t)c * Df + d];
        all[c] = {tn[c] > 0.0 ? s / tn[c] : 0.0, c};
      }
      std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
      });
      ids[n] = kv.first;
      for (int32_t i = 0; i < kk; ++i) {
        classes[n * kk + i] = all[i].second;
        scores[n * kk + i] = all[i].first;
      }
    }
    n++;
  }
  return n;
}

/* dense transfer (NEXT f4): P:201 [§IV-B] "associating each 3D point in the ground truth to its */
/* closest CLIP feature vector in our mapped scene"; "each gt point takes the top-1   */
/* class of the spatially nearest instance (nearest voxel center over all instances); points     */
/* farther than d_assign from any voxel labeled unassigned".  R40: distance to the voxel centre  */
/* (k + 0.5) r, squared, in fp64 with r = (double)voxel_size, point coordinates fp32 promoted,   */
/* summed x, y, z in that order; the minimum (d^2, id) wins (ties: lower id); unassigned  */
/* iff d^2 > d_assign^2 (fp64).  Brute force over the membership relation.                        */
extern "C" void ora_dense_transfer(const ora_map* m, const float* pts, int64_t P, float d_assign, int64_t* out) {
  const double r = (double)m->cfg.voxel_size, dmax = (double)d_assign * (double)d_assign;
  for (int64_t p = 0; p < P; ++p) {
    double best = INFINITY;
    Id bid = -1;
    for (const auto& kv : m->mem) {
      double d2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const double c = ((double)kv.first[a] + 0.5) * r;
        const double x = (double)pts[3 * p + a] - c;
        d2 = d2 + x * x;
      }
      for (Id j : kv.second)
        if (d2 < best || (d2 == best && j < bid)) { best = d2; bid = j; }
    }
    out[p] = (bid >= 0 && best <= dmax) ? bid : -1;
  }
}
