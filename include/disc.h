/*
 * disc.h -- C ABI of libdisc, the B200-native (sm_100a) DISC per-frame mapping hot path.
 *
 * DISC (arXiv 2603.03935) §III: each frame's instance masks are back-projected through
 * depth and pose into voxel keys, hashed into a GPU-resident voxel map, the exact
 * voxel overlap of every new segment with the map's instances is counted,
 * instances are associated / merged on the fly when overlap and visual similarity suffice
 * (P:98), and dense ViT patch tokens are pooled under each mask weighted by the
 * distinctiveness map D (Eq.1) into per-instance embeddings that are replaced on
 * fusion by the observation of higher quality Q (Eq.2-3).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; R<k> = reading k in DESIGN.md §3
 * (SURVEY.md §8(c) C.3).  The operation a call performs is defined step by step in
 * DESIGN.md §2 (= SURVEY §8(c) C.2, O0-O13).
 *
 * Conventions
 *  - Plain C, no CUDA types: a stream is passed as `void*` (a cudaStream_t; NULL = legacy
 *    default stream).  Device pointers are CUDA device addresses on the map's device.
 *  - Ownership: the caller owns every input buffer; device inputs must stay valid until the
 *    work enqueued on `stream` completes (stream-ordered, as in cuBLAS).  The library owns
 *    all map state (device memory allocated in disc_map_create, freed in destroy).
 *    Outputs go to caller-allocated HOST buffers.  Getters called with NULL output
 *    buffers return the required count in *n_out; a short `cap` returns DISC_ERR_INVALID.
 *  - Errors: argument / frame validation failures return DISC_ERR_INVALID before any
 *    mutation (non-rigid pose S:118, dims, capacities, thresholds S:320).  Per-segment
 *    problems never fail a frame; they are counted in the report by reason.
 *    Capacity, CUDA and internal errors are sticky: the map is poisoned, later calls
 *    return the same code, disc_last_error() gives the text.  Capacity overflow detected on
 *    the device is reported at the next synchronising call (one that fills a host buffer).
 *  - Threading: one writer per map.  Query / get calls must not run concurrently
 *    with integrate calls on the same map.
 *  - No CPU fallback: every step of the path runs in libdisc's sm_100a kernels.
 */
#ifndef DISC_H
#define DISC_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DISC_OK = 0,
  DISC_ERR_INVALID = 2,      /* bad argument / frame / config; nothing was mutated        */
  DISC_ERR_INTERNAL = 4,
  DISC_ERR_CAPACITY = 5,     /* a configured capacity was exceeded (sticky)               */
  DISC_ERR_CUDA = 6,         /* CUDA runtime error (sticky)                               */
  DISC_ERR_NCCL = 7,
  DISC_ERR_UNSUPPORTED = 8
} disc_status;

typedef struct disc_map disc_map;  /* opaque, library-owned */

typedef struct {
  /* method parameters */
  float voxel_size;        /* r (m) > 0        */
  float tau_geo;           /* overlap_min threshold in (0,1], default 0.3   R10, S:356       */
  float tau_vis;           /* tracking cosine threshold in [-1,1], 0.8      R11, R15  */
  float depth_min, depth_max;        /* exclusive validity window 0.1/10  R4 */
  float mask_min_conf;     /* 0.5                                           R8        */
  float mask_max_aspect;   /* 10 (long/short bbox side, inclusive)          R8        */
  int32_t mask_min_area;   /* 400 pixels (inclusive)                        R8        */
  float cover_min;         /* 0.25 (patch coverage threshold, inclusive)   R17, R18  */
  float lambda_size;       /* 3.3            */
  float eps_distinct;      /* 1e-6                                          Eq.1, R16        */
  float dbscan_eps;        /* > 0: DBSCAN denoise of each segment's points before voxelisation */
                           /* (R42): the largest cluster is kept; 0 = off (R7) */
  int32_t dbscan_min_pts;  /* core threshold (points within eps, the point included), >= 1      */
  int32_t refine_active;   /* 1: after each frame's update, instance pairs of the frame's active   */
                           /* set that pass the same test merge, to a fixpoint (S:327 step (3),    */
                           /* P:98 "among all candidates"; R43); 0 = off (R14)                     */
  int32_t feat_dim;        /* Df in [4,1024], multiple of 4 (CLIP token width)               */
  int32_t track_dim;       /* Dt in [0,512]; 0 = no visual gate (DINO tracking width)        */
  /* capacities (device memory is sized from these at create time) */
  int64_t max_memberships; /* live (key, instance) pairs; voxel hash sized 2x               */
  int32_t max_instances;   /* instance ids ever created (ids are never reused, R13)          */
  int32_t max_masks;       /* S per frame, <= 255                                            */
  int32_t max_pixels;      /* H*W per frame                                                  */
  int32_t max_patches;     /* Hp*Wp per frame                                                */
  int32_t max_pairs_per_frame; /* unique (mask, voxel) pairs per frame (all masks, dropped  */
                               /* ones included), <= 2^22; a frame past it fails with the   */
                               /* sticky DISC_ERR_CAPACITY.  Also sizes the frame hash      */
                               /* tables (2x, power of two) and the per-frame item list     */
                               /* between the mask pass and the dedup (an overflowing list  */
                               /* falls back to direct inserts, never to an error)          */
  int32_t window;          /* frames per stage-1 batch in disc_integrate_frames, 1..32       */
  int32_t device;          /* CUDA ordinal                                                   */
  /* key-hash sharding: world_size = G shards; shard g owns the    */
  /* voxel keys with (mix64(key) >> 40) mod G == g (memberships, hash slots, key lists) and a   */
  /* replica of the instance table.  G = 1: unsharded (rank 0, nccl_unique_id NULL).            */
  /* G > 1, nccl_unique_id == NULL: all G shards in this process on `device` (exchanges =       */
  /*   device copies; rank must be 0; G <= 16); the caller passes the whole frame stream.       */
  /* G > 1, nccl_unique_id = the 128 bytes of disc_nccl_unique_id() created by rank 0 and       */
  /*   broadcast out of band: this process is shard `rank` of G (one GPU each, NCCL exchanges   */
  /*   on the caller's stream).  Every rank calls the same sequence of integrate calls, each    */
  /*   with the SAME number of its own frames: rank r's j-th frame is frame r + G j of the      */
  /*   stream (windows of floor(window / G) frames per rank).  Reports are returned for the     */
  /*   caller's own frames; the instance table is replicated and bit-identical to G = 1;       */
  /*   disc_get_memberships returns this process's shards' keys.                                */
  int32_t world_size, rank;
  const void* nccl_unique_id;
} disc_config;

typedef struct {
  int64_t frame_id;
  int32_t height, width;               /* H_img, W_img                                      */
  float fx, fy, cx, cy;                /* pinhole intrinsics; pixel (u,v) integer (R1)       */
  float pose[16];                      /* camera->world, row-major, OpenCV axes (R3); host   */
  const float* depth;                  /* [H][W] z-depth, metres (R2)                        */
  int32_t num_masks;                   /* S >= 0                                             */
  const uint8_t* masks;                /* [S][H][W], nonzero = in mask (R9: may overlap)     */
  const float* mask_conf;              /* [S] or NULL (= 1.0)                                */
  int32_t patch_h, patch_w;            /* Hp in [1,H], Wp in [1,W]; pixel -> patch by floor  */
                                       /* (v Hp / H, u Wp / W) (R17)                         */
  const float* patch_feats;            /* [Hp][Wp][Df] fp32 CLIP tokens, or NULL: geometry-  */
                                       /* only mode (no embedding, Q = -1)                   */
  const float* global_embed;           /* [Df] or NULL (S_sem = 1)                           */
  const uint16_t* track_feats;         /* [Hp][Wp][Dt] bf16 bit patterns; required iff Dt>0  */
  const uint32_t* mask_bits;           /* the masks bit-packed, instead of `masks` (exactly  */
                                       /* one of the two non-NULL when S > 0): plane s is    */
                                       /* ceil(H*W/32) little-endian words, pixel p = v*W+u  */
                                       /* is bit p%32 of word p/32 (bits past H*W ignored);  */
                                       /* 1/8 of the bytes to move and to read   */
} disc_frame;

typedef struct {                       /* per-frame report                     */
  int32_t kept, drop_area, drop_conf, drop_aspect, drop_nodepth, drop_nofeat;
  int64_t key_out_of_range;            /* depth-valid pixels with a key outside +-2^20 (R6) */
  int64_t unique_pairs;                /* U = sum over kept s of |V_s|                      */
  int64_t edges;                       /* qualifying (s, j) edges (O10)                     */
  int64_t created, merged_away;
  int64_t new_memberships;             /* net growth of the membership relation             */
  int64_t relabeled;                   /* sum of |V_j| over merged-away instances j         */
  int64_t live_instances, live_memberships;
  int64_t refine_rounds;               /* refine_active: rounds of instance-pair merges (R43) */
  int64_t refine_merged;               /* refine_active: instances merged away by them        */
} disc_frame_report;

typedef struct {
  int64_t id, voxel_count, last_seen;
  int32_t obs_count;
  float q;                             /* quality of the kept embedding; -1 = none          */
  int32_t aabb_min[3], aabb_max[3];    /* key-space bounds of the voxel set                  */
} disc_instance;

typedef struct {                       /* last-frame debug export (parity tests)            */
  int32_t num_masks;                   /* out                                                */
  int32_t* status;                     /* [S] 0 kept,1 area,2 conf,3 aspect,4 nodepth,5 nofeat */
  int64_t* area;                       /* [S]                                                */
  int32_t* bbox;                       /* [S][4] umin, vmin, umax, vmax                      */
  int64_t* vs;                         /* [S] |V_s|                                          */
  int64_t* target;                     /* [S] instance id the detection was fused into, -1   */
  float* factors;                      /* [S][6] s_size, s_angle, s_sem, s_dist, q, dbar     */
  float* embed;                        /* [S][Df] e_s                                        */
  double* track;                       /* [S][Dt] t_s                                        */
  int64_t pair_cap;                    /* capacity of pair_s / pair_key                      */
  int32_t* pair_s;                     /* unique (s, key) pairs of kept detections, any order */
  uint64_t* pair_key;                  /* packed keys (R6)                                    */
  int64_t n_pairs;                     /* out                                                */
  int64_t trip_cap;
  int32_t* trip_s;                     /* C triples (s, j, c) over kept s, frame-start j      */
  int64_t* trip_j;
  int64_t* trip_c;
  int32_t* trip_edge;
  int64_t n_trip;                      /* out                                                */
} disc_frame_debug;

typedef struct {                       /* timing of the dominant kernels (disc_set_timing)  */
  int64_t frames;
  double k1_ms;                        /* mask pass + back-projection + dedup (K1)          */
  int64_t k1_launches;
  double stage1_ms, stage2_ms;         /* whole stage-1 batch / sum of stage-2 frame loops  */
  int64_t mask_bytes, depth_bytes, track_bytes, feat_bytes; /* algorithmic input bytes      */
  int64_t pairs, map_inserts, relabels; /* sum U, labels inserted, relabel items processed    */
  int64_t edges;                       /* sum of qualifying (s, j) edges                     */
  int64_t launches;                    /* kernels launched by integrate calls                */
  int64_t shard_memberships[16];       /* live memberships held by each shard of this process */
                                       /* (sharded map: the keys it owns; unsharded: [0] all) */
} disc_stats;

typedef struct {                       /* disc_finalize report                                */
  int64_t rounds;                      /* union-find rounds that merged something (R35)      */
  int64_t edges;                       /* qualifying instance pairs, summed over the rounds  */
  int64_t merged_away;                 /* instances erased by merges                          */
  int64_t relabeled;                   /* sum of |V_j| over merged-away instances j           */
  int64_t removed;                     /* instances below min_voxels (R38)                    */
  int64_t live_instances, live_memberships;
} disc_final_report;

/* Fill *c with the defaults named above (capacities sized for a Replica-shaped stream). */
disc_status disc_config_init(disc_config* c);
disc_status disc_map_create(const disc_config* cfg, disc_map** out);
void disc_map_destroy(disc_map* m);

/* One frame, device-resident inputs (O0-O13).  report (host) may be NULL; a non-NULL
 * report synchronises.  On return `stream` is ordered after the last read of the caller's
 * inputs; the map update itself may still be running on the library's internal stage-2 stream
 * (so the next call's per-frame stage 1 overlaps it).  disc_wait orders a stream after all of
 * the map's work; every reader (query / get / debug / sync) waits for it. */
disc_status disc_integrate_frame(disc_map* m, const disc_frame* f, void* stream,
                                 disc_frame_report* report);
/* == n sequential disc_integrate_frame calls; batches stage 1 (per-frame independent work)
 * over windows of cfg.window frames.  report: host array [n] or NULL. */
disc_status disc_integrate_frames(disc_map* m, const disc_frame* f, int32_t n, void* stream,
                                  disc_frame_report* report);
/* Same, but every data pointer of f[i] is HOST memory (pinned for full speed): the
 * library copies each window's inputs to device staging buffers on `stream`. */
disc_status disc_integrate_frames_host(disc_map* m, const disc_frame* f, int32_t n, void* stream,
                                       disc_frame_report* report);

/* Q1: top-k live instances by cosine e_j . q/|q|, ties by ascending id.
 * q: host [Df]; ids/scores: host [k]; synchronises. */
disc_status disc_query(disc_map* m, const float* q, int32_t k, int64_t* ids, float* scores,
                       int32_t* n_out);
/* Q2: live instances, ascending id; embeds host [cap][Df] or NULL; track host [cap][Dt] or
 * NULL (fp64 sums T_j, R15). */
disc_status disc_get_instances(disc_map* m, disc_instance* out, float* embeds, double* track,
                               int32_t cap, int32_t* n_out);
/* membership relation {(key, id)} (any order); keys packed per R6. */
disc_status disc_get_memberships(disc_map* m, uint64_t* keys, int64_t* ids, int64_t cap,
                                 int64_t* n_out);
disc_status disc_debug_last_frame(disc_map* m, disc_frame_debug* d);
/* End of trajectory (P:100 [§III-B]: "merge remaining orphaned candidates and filter out residual
 * noisy instances, such as segments containing fewer than a minimum threshold of voxels";
 * S:333-337; readings R35-R38): every pair of live instances (i < j) with c_ij = |V_i ∩ V_j| >= 1,
 * c_ij >= tau_geo min(|V_i|, |V_j|) (exact) and, when Dt > 0, (dot_pin(T_i,T_j) / sqrt(dot_pin(T_i,T_i)))
 * / sqrt(dot_pin(T_j,T_j)) >= tau_vis is an edge; components merge into their min id (T summed in
 * ascending id order, (e, Q) replaced iff strictly higher in that order, obs summed, last_seen =
 * max); repeated until no pair qualifies; then every instance with |V| < min_voxels is removed with
 * its memberships.  Pass the map's own tau_geo / tau_vis for SPEC's finalize.  Synchronises; the
 * map stays usable (integration may continue).  DISC_ERR_UNSUPPORTED on a sharded map. */
disc_status disc_finalize(disc_map* m, float tau_geo, float tau_vis, int64_t min_voxels, disc_final_report* rep);
/* NEXT f4, batched open-vocabulary retrieval (P:195 [§IV-A] "top-k cosine-similarity predictions";
 * S:398-403; R39): for every live instance with an embedding (ascending id) the k (1..16) best rows
 * of table (host [C][Df], class text embeddings in the token space, R23) by cos = e_j . t_c / |t_c|,
 * descending, ties by ascending class index.  ids host [cap], classes / scores host [cap][min(k,C)];
 * NULL ids: count only.  Synchronises. */
disc_status disc_classify(disc_map* m, const float* table, int32_t C, int32_t k, int64_t* ids, int32_t* classes,
                          float* scores, int64_t cap, int64_t* n_out);
/* NEXT f4, dense transfer (P:201 [§IV-B]; R40): for each point (host [P][3], world metres)
 * the id of the instance owning the nearest voxel centre (k + 0.5) r (ties: lower id), or -1 when
 * that centre is farther than d_assign (<= 64 voxels).  out host [P].  DISC_ERR_UNSUPPORTED on a
 * sharded map.  Synchronises. */
disc_status disc_dense_transfer(disc_map* m, const float* points, int64_t P, float d_assign, int64_t* out);
disc_status disc_set_timing(disc_map* m, int32_t on);
disc_status disc_get_stats(disc_map* m, disc_stats* s);
disc_status disc_wait(disc_map* m, void* stream);  /* order `stream` after all queued map work */
disc_status disc_sync(disc_map* m);    /* wait for the map's work; surfaces device errors */
const char* disc_last_error(const disc_map* m);
const char* disc_version(void);
/* NCCL unique id for the key-sharded map: 128 bytes that rank 0 creates
 * and broadcasts out of band; every rank then passes it in disc_config.nccl_unique_id.  Loads
 * libnccl.so.2 at run time; DISC_ERR_NCCL if it is missing or fails. */
disc_status disc_nccl_unique_id(uint8_t out[128]);

#ifdef __cplusplus
}
#endif
#endif
