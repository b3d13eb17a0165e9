// disc_launch.h -- host-side launchers of libdisc's kernels (internal).
#pragma once
#include "disc_common.cuh"

namespace disc {
// DISC_DEBUG_SYNC=1: synchronise and check after every launch, naming the kernel (debugging
// aid for device faults; off by default).
void debug_check(cudaStream_t st, const char* kernel, int frame);
void k6_prof_dump();
int k1_nsmid();   // %nsmid of the current device (upper bound of %smid)
size_t k6_smem_bytes(int S, int TC);
size_t k6_layout_bytes(int S, int TC);   // the association's table layout alone (global-memory mode)
int launch_stage1(const WinDesc& wd, const WinBufs& wb, const Params& P, int* err, bool sem, int maxS,
                  int maxHp, int maxW, int maxWp, int maxP, int rows_cap, int nsm, int nres, cudaStream_t st,
                  cudaEvent_t ev0, cudaEvent_t ev1, bool fill_ktab = true, bool fill_nsum = true,
                  bool release = false);
void launch_refine(int f, int S, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P, int grid,
                   cudaStream_t st);
int launch_stage2(const WinDesc& wd, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P,
                  bool sem, int nsm, int nres, uint32_t* tag_seq, int spec_mode, cudaStream_t st);
// NEXT f3 (k_dbscan.cu): DBSCAN denoise replacing K1b / K1c when P.db_eps > 0; returns launches
int launch_dbscan(const WinDesc& wd, const WinBufs& wb, const Params& P, int* err, bool sem, int nsm, cudaStream_t st);
size_t dbscan_tmp_bytes(int n_items, int n_seg);
// the key-hash-sharded map (k_map.cu: stage-2 phases per frame; k_shard.cu: stage-1 exchange)
// phase 0 lookup, 1 association (one CTA), 2 apply
void launch_stage2_sharded_frame(int phase, int f, const FrameMeta* meta, const WinBufs& wb, const MapState& M,
                                 const FrameScratch& X, const Params& P, bool sem, int grid, cudaStream_t st);
void launch_trip_pack(const FrameScratch& X, uint32_t* out, int cap, int* err, cudaStream_t st);
void launch_trip_merge(const FrameScratch& X, const uint32_t* all, size_t stride, int G, int self, int* err,
                       cudaStream_t st);
void launch_add_pack(const MapState& M, const FrameScratch& X, int64_t* out, int smax, cudaStream_t st);
void launch_finalize_sum(int f, const MapState& M, const FrameScratch& X, const int64_t* all, int parts, size_t stride,
                         int smax, cudaStream_t st);   // all: [parts][stride] rows summed
struct DetLayout {   // one frame's detection records, replicated to every shard (bytes)
  size_t status, vs, qf, tok, daabb, area, bbox, emb, trk, meta, total;
  DetLayout(int SMAX, int Df, int Dt) {
    size_t o = 0;
    auto take = [&](size_t b) { const size_t r = o; o = (o + b + 15) & ~(size_t)15; return r; };
    meta = take(32);   // S, frame_id, key_out_of_range
    status = take(4 * (size_t)SMAX); vs = take(4 * (size_t)SMAX); qf = take(24 * (size_t)SMAX);
    tok = take((size_t)SMAX); daabb = take(24 * (size_t)SMAX); area = take(4 * (size_t)SMAX);
    bbox = take(16 * (size_t)SMAX); emb = take(4 * (size_t)SMAX * Df); trk = take(8 * (size_t)SMAX * (Dt > 0 ? Dt : 1));
    total = o;
  }
};
struct PairRec { unsigned long long key; uint32_t info; uint32_t pad; };   // info = frame slot << 8 | s
constexpr int MAX_LOCAL_SHARDS = 16;
struct RouteDst {   // destination shards' stage-2 pair arrays (shards of one process, same device)
  unsigned long long* pkey[MAX_LOCAL_SHARDS];
  uint32_t* pinfo[MAX_LOCAL_SHARDS];
  uint32_t* npairs[MAX_LOCAL_SHARDS];
  int32_t PMAX;
};
// pack this shard's stage-1 frames (local slots 0..n-1; meta per frame) into det records
void launch_det_pack(const WinBufs& src, int n, const FrameMeta* meta_host, uint8_t* buf, const DetLayout& L, int Df,
                     int Dt, bool sem, cudaStream_t st);
// unpack window slot i = r + G j from buf[(r * nloc + j)] into dst slot i; meta_dst[i] too
void launch_det_unpack(const uint8_t* buf, int n, int G, int nloc, const DetLayout& L, const WinBufs& dst,
                       FrameMeta* meta_dst, int Df, int Dt, bool sem, cudaStream_t st);
// route the kept detections' unique (s, key) pairs of this shard's frames (local slot j = window
// slot g + G j) to their owners: direct delivery into dst (one process), or counting (counts[G])
// then scattering into send (offsets[G]) for an NCCL exchange
void launch_pair_route(const WinBufs& src, int n, int g, int G, const RouteDst* dst, unsigned long long* counts,
                       const unsigned long long* offsets, PairRec* send, int* err, cudaStream_t st);
void launch_pair_deliver(const PairRec* recv, unsigned long long n, const WinBufs& dst, int* err, cudaStream_t st);

// disc_finalize (k_final.cu): rep_out = rounds, edges, merged_away, relabeled, removed, live_instances,
// live_memberships
int run_finalize(const MapState& M, int Df, int Dt, int64_t next_id, float tau_geo, float tau_vis, int64_t min_voxels,
                 int* err, cudaStream_t st, int64_t rep_out[7]);
// export / query
int64_t export_instances(const MapState& M, int Df, int Dt, int64_t next_id, disc_instance* out,
                         float* embeds, double* track, int32_t cap, cudaStream_t st, void* scratch,
                         size_t scratch_bytes);
int64_t export_memberships(const MapState& M, uint64_t* keys, int64_t* ids, int64_t cap, cudaStream_t st,
                           void* scratch, size_t scratch_bytes);
int64_t run_classify(const MapState& M, int Df, int64_t next_id, const float* table_host, int32_t C, int32_t k,
                     int64_t* ids_out, int32_t* cls_out, float* sc_out, int64_t cap, cudaStream_t st, void* scratch,
                     size_t scratch_bytes);
int run_dense_transfer(const MapState& M, float r, const float* pts_host, int64_t P, float d_assign, int64_t* out_host,
                       cudaStream_t st, void* scratch, size_t scratch_bytes);
void slot_stats(const MapState& M, cudaStream_t st);   // DISC_SLOT_STATS diagnostic
int32_t run_query(const MapState& M, int Df, int64_t next_id, const float* q_host, int32_t k, int64_t* ids,
                  float* scores, cudaStream_t st, void* scratch, size_t scratch_bytes);
}  // namespace disc
