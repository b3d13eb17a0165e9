/*
 * disc_oracle.h -- C API of the CPU oracle for the DISC per-frame mapping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the slow, definitional reference that
 * the CUDA path (paper_2603_03935_b200/) is checked against.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or helper with the CUDA path.
 *
 * Citations:  P:n = /root/reference/PAPER.md line n,  S:n = /root/reference/SPEC.md
 * line n, R<k> = reading k of SURVEY.md §8(c) C.3 (restated in DESIGN.md §3).
 *
 * Layouts (all row-major, host memory, caller-owned):
 *   depth       float [H][W]        z-depth in metres (R2)
 *   masks       uint8 [S][H][W]     values {0,1}
 *   mask_conf   float [S] or NULL   (NULL = 1.0)
 *   patch_feats float [Hp][Wp][Df]  or NULL = geometry-only mode
 *   global_embed float [Df] or NULL (S_sem = 1)
 *   track_feats uint16 [Hp][Wp][Dt] bf16 bit patterns, required iff track_dim > 0
 *   pose        float [16] camera->world, row-major, OpenCV camera axes (R3)
 */
#ifndef DISC_ORACLE_H
#define DISC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float voxel_size;        /* r > 0 (m) */
  float tau_geo;           /* (0,1]                              R10       */
  float tau_vis;           /* [-1,1]                             R11, R15  */
  float depth_min, depth_max;                   /* exclusive    R4        */
  float mask_min_conf, mask_max_aspect;         /*              R8        */
  int32_t mask_min_area;
  float cover_min;         /* 0.25                               R17, R18  */
  float lambda_size;       /* 3.3     */
  float eps_distinct;      /* 1e-6                               R16       */
  float dbscan_eps;        /* > 0: DBSCAN denoise (R42), metres; 0 = off (R7) */
  int32_t dbscan_min_pts;  /* core threshold, neighbours incl. the point itself     */
  int32_t refine_active;   /* 1: per-frame instance x instance refinement (S:327 (3), R43) */
  int32_t feat_dim;        /* Df > 0                                       */
  int32_t track_dim;       /* Dt >= 0, 0 = no visual gate                  */
} ora_config;

typedef struct {
  int64_t frame_id;
  int32_t height, width;
  float fx, fy, cx, cy;
  float pose[16];
  const float* depth;
  int32_t num_masks;
  const uint8_t* masks;
  const float* mask_conf;
  int32_t patch_h, patch_w;
  const float* patch_feats;
  const float* global_embed;
  const uint16_t* track_feats;
} ora_frame;

typedef struct {
  int32_t kept, drop_area, drop_conf, drop_aspect, drop_nodepth, drop_nofeat;
  int64_t key_out_of_range;  /* depth-valid pixels whose key is outside [-2^20,2^20) (R6) */
  int64_t unique_pairs;      /* U = sum over kept s of |V_s|                               */
  int64_t edges;             /* |E| (O10)                                                  */
  int64_t created;           /* new instance ids                                           */
  int64_t merged_away;       /* instances erased by merges                                 */
  int64_t new_memberships;   /* net growth of the membership relation this frame           */
  int64_t relabeled;         /* sum of |V_j| over merged-away instances j                  */
  int64_t live_instances, live_memberships;
  int64_t refine_rounds;     /* refine_active: union-find rounds that merged instance pairs     */
  int64_t refine_merged;     /* refine_active: instances merged away by the refinement          */
} ora_report;

/* mask status codes (O1, O3, O7) */
enum { ORA_KEPT = 0, ORA_DROP_AREA = 1, ORA_DROP_CONF = 2, ORA_DROP_ASPECT = 3,
       ORA_DROP_NODEPTH = 4, ORA_DROP_NOFEAT = 5 };
/* return codes */
enum { ORA_OK = 0, ORA_INVALID = 2, ORA_SELFCHECK_FAILED = 4 };

typedef struct ora_map ora_map;

ora_map* ora_create(const ora_config* cfg);          /* NULL on invalid config */
void     ora_destroy(ora_map* m);
void     ora_set_selfcheck(ora_map* m, int32_t on);  /* brute-force cross-checks inside integrate */
int32_t  ora_integrate(ora_map* m, const ora_frame* f, ora_report* rep);
const char* ora_last_error(const ora_map* m);

/* finalize (readings R35-R38): orphan merge to a fixpoint, then the minimum-
   size filter.  Thresholds are explicit (pass the map's own tau_geo / tau_vis for SPEC's op). */
typedef struct {
  int64_t rounds;            /* union-find rounds that merged something                         */
  int64_t edges;             /* qualifying instance pairs, summed over the rounds               */
  int64_t merged_away;       /* instances erased by merges                                      */
  int64_t relabeled;         /* sum of |V_j| over merged-away instances                         */
  int64_t removed;           /* instances below min_voxels                                      */
  int64_t live_instances, live_memberships;
} ora_final_report;
int32_t  ora_finalize(ora_map* m, float tau_geo, float tau_vis, int64_t min_voxels, ora_final_report* rep);

/* batched retrieval (R39): top-k classes of every live instance with an
   embedding, ascending id; classes / scores [n][min(k, C)]; returns n (fills at most cap rows) */
int64_t ora_classify(const ora_map* m, const float* table, int32_t C, int32_t k, int64_t* ids,
                     int32_t* classes, double* scores, int64_t cap);
/* dense transfer (R40): nearest-voxel-centre instance of each point [P][3]
   (world, metres), -1 if farther than d_assign */
void    ora_dense_transfer(const ora_map* m, const float* pts, int64_t P, float d_assign, int64_t* out);

/* P:92 / S:123-131 DBSCAN (R42): the classic sequential algorithm over points [n][3] (fp32, taken
   in index order), squared distances in fp64 (dx^2 + dy^2 + dz^2, no contraction) against
   (double)eps^2, a point's neighbourhood including itself; labels[i] = cluster number in creation
   order (0, 1, ...) or -1 (noise); returns the number of clusters */
int32_t ora_dbscan(int64_t n, const float* pts, float eps, int32_t min_pts, int32_t* labels);

/* ---- map state export ---- */
int64_t ora_num_instances(const ora_map* m);
/* ascending id; e [n][Df] (zeros if q == -1), T [n][Dt]; any pointer may be NULL */
int64_t ora_get_instances(const ora_map* m, int64_t* id, int64_t* vcount, int32_t* obs,
                          int64_t* last_seen, double* q, int32_t* aabb6, double* e,
                          double* T, int64_t cap);
int64_t ora_num_memberships(const ora_map* m);
/* sorted by (packed key, id) */
int64_t ora_get_memberships(const ora_map* m, uint64_t* keys, int64_t* ids, int64_t cap);
/* R22 acceptance set of instance id: observations with q >= qmax*(1-1e-4) */
int64_t ora_get_accept(const ora_map* m, int64_t id, double* q, double* e, int64_t cap);
int64_t ora_next_id(const ora_map* m);

/* ---- last-frame debug export (state of the most recent ora_integrate) ---- */
int32_t ora_last_num_masks(const ora_map* m);
/* per mask s: status, area, bbox (umin,vmin,umax,vmax), |V_s|, target id (-1 if not kept) */
void    ora_last_masks(const ora_map* m, int32_t* status, int64_t* area, int32_t* bbox4,
                       int64_t* vs, int64_t* target);
/* unique (s,key) pairs of kept detections, sorted by (s, key) */
int64_t ora_last_pairs(const ora_map* m, int32_t* s, uint64_t* keys, int64_t cap);
/* C triples (s, j, c>0) over kept s and frame-start live j, sorted by (s,j); edge flag */
int64_t ora_last_triples(const ora_map* m, int32_t* s, int64_t* j, int64_t* c, int32_t* edge,
                         int64_t cap);
/* factors [S][6] = s_size, s_angle, s_sem, s_dist, q, dbar; e [S][Df]; u,t [S][Dt] */
void    ora_last_quality(const ora_map* m, double* factors6, double* e, double* u, double* t);

/* ---- single steps, exported for the pin tests ---- */
/* O2: world point of pixel (u,v) by the pinned fp32 formula (R5); returns 1 iff depth valid */
int32_t ora_pixel_world(const ora_config* c, const ora_frame* f, int32_t u, int32_t v,
                        float out[3]);
/* O2: key = floor(p / r) in fp32 (R5); returns 1 iff every component in [-2^20, 2^20) */
int32_t ora_point_key(const float p[3], float r, int32_t out[3]);
uint64_t ora_pack_key(int32_t ix, int32_t iy, int32_t iz);   /* R6 */
/* A0: pose rigidity */
int32_t ora_pose_rigid(const float pose[16]);
/* O6 / Eq.1: D[P] from feats [P][Df] */
void    ora_distinctiveness(int64_t P, int32_t Df, const float* feats, double eps, double* D);
/* O7 pooling for one mask: cnt[P], npix[P], D[P], feats[P][Df] -> e[Df], dbar; returns
   0 ok, 1 zero vector ("nofeat") */
int32_t ora_pool(int64_t P, int32_t Df, const int64_t* cnt, const int64_t* npix,
                 const double* D, const float* feats, double cover_min, double* e,
                 double* dbar);
double  ora_s_size(int64_t area, int32_t H, int32_t W, double lambda);
/* Eq.3 over n voxels: unit normals [n][3], unit rays [n][3] */
double  ora_s_angle(int64_t n, const double* normals, const double* rays);
double  ora_s_sem(int32_t Df, const double* e, const float* g);
double  ora_s_dist(double dbar);
double  ora_quality(double s_size, double s_angle, double s_sem, double s_dist);
/* R15 pinned fp64 dot: 32 lane partials (fma, ascending), xor butterfly 16,8,4,2,1 */
double  ora_dot_pin(int32_t n, const double* a, const double* b);
/* query (Q1): scores of live instances vs q/|q|, full sort, ties by ascending id */
int64_t ora_query(const ora_map* m, const float* q, int32_t k, int64_t* ids, double* scores);

#ifdef __cplusplus
}
#endif
#endif
