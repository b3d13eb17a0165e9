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
                  cudaEvent_t ev0, cudaEvent_t ev1);
int launch_stage2(const WinDesc& wd, const WinBufs& wb, const MapState& M, const FrameScratch& X, const Params& P,
                  bool sem, int nsm, int nres, cudaStream_t st);
// export / query
int64_t export_instances(const MapState& M, int Df, int Dt, int64_t next_id, disc_instance* out,
                         float* embeds, double* track, int32_t cap, cudaStream_t st, void* scratch,
                         size_t scratch_bytes);
int64_t export_memberships(const MapState& M, uint64_t* keys, int64_t* ids, int64_t cap, cudaStream_t st,
                           void* scratch, size_t scratch_bytes);
int32_t run_query(const MapState& M, int Df, int64_t next_id, const float* q_host, int32_t k, int64_t* ids,
                  float* scores, cudaStream_t st, void* scratch, size_t scratch_bytes);
}  // namespace disc
