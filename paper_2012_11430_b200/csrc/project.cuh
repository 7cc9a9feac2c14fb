// project.cuh — host/device interface of the projection kernels (project.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace prony {

int64_t ext_rows(int d, int n);  // |E| = (n+2)^d
constexpr int kPtabPad = 4;   // P table padded so the last k-step may read P(h) for h < N+4
constexpr int kMaxNP = 128;   // padded width of Y rows handled by k_reduce
constexpr int kYCap = 4;      // split-K bound: KC * (rows in range) <= kYCap * d * N
#ifndef PRONY_BK
#define PRONY_BK 16
#endif
#ifndef PRONY_STAGES
#define PRONY_STAGES 3
#endif
constexpr int kBK = PRONY_BK;          // columns of T_l per pipeline stage of k_project (8 or 16)
constexpr int kStages = PRONY_STAGES;  // cp.async ring depth of k_project (<= 227 KB smem)
static_assert(kBK == 8 || kBK == 16, "stage width: 8 or 16 columns (the P(h) lanes and B-row lanes)");

struct ProjShape {
  int NT, WN, WM, BM;  // k_project consumer layout
  int rNT, rWN, BI;    // k_reduce layout
  int NP;
};

// rows of T_l covered by a call: for l = 1..d (index l-1), rows [kb, kb+rows) of I_n.
// shared = 1 (PRONY_UNITS_SHARED): the call covers rows [e0, e1) of the extended block
// T_E = [f(k'-h)], k' in E = {0..n+1}^d (lexicographic, last fastest), and every S_l takes its rows
// from the same product: T_l[k,:] = T_E[k+e_l,:] (F8), so k_project runs once for all l.
struct ProjGeom {
  int d, n, m, N;
  int kb[PRONY_MAX_D];
  int rows[PRONY_MAX_D];
  int shared;
  int e0, e1;
};

struct ProjPlan {
  ProjShape shape;
  int yoff[PRONY_MAX_D];
  int R_tot, max_rows;
  int chunk_w, KC;  // split-K: KC chunks of chunk_w columns of T_l (chunk 0: chunk0_w columns)
  int chunk0_w;     // width of chunk 0 (= chunk_w, or narrower after project_plan_lead)
  int RP;           // reduce partitions per l (the largest over the j-blocks)
  int nj;           // j-blocks of the warp-specialized reduce (k_reduce_ws)
  int rp_j[4];      // its row partitions per j-block (weighted by the j-block's active m-tiles)
};

struct ProjParams {
  const double2* grid;
  const double* gsum;
  const double2* V;
  int ldv;  // row stride of V (elements)
  const double* vsum;
  const int32_t* ptab;
  const int32_t* rtab;  // row table: ptab (per-l rows of I_n) or etab (rows of E, shared mode)
  double2* Y;
  int* counters;  // [d][nrb] split-K arrival counters (zeroed per call)
  int N, m, NP, chunk_w, R_tot, KC, nrb;
  int chunk0_w;  // chunk c covers columns [c ? chunk0_w + (c-1) chunk_w : 0, +width) of T_l
  int box;  // grid size (debug index checks)
  int chunk_base;  // first split-K chunk of this launch (blockIdx.y + chunk_base)
  int kb[PRONY_MAX_D], rows[PRONY_MAX_D], yoff[PRONY_MAX_D], shift[PRONY_MAX_D];
};

struct RedParams {
  const double2* Y;
  const double2* U;
  const int32_t* umap;  // shared mode: umap[l*E + e] = row of U paired with row e of Y_E for S_l, or -1
  double2* Spart;
  int m, NP, KC, R_tot, RP, E;
  int kb[PRONY_MAX_D], rows[PRONY_MAX_D], yoff[PRONY_MAX_D];
  int rp_j[4];  // k_reduce_ws: row partitions of j-block z (CTAs with blockIdx.x >= rp_j[z] write zeros)
};

// Copy/compute overlap for callers whose V arrives in pieces (prony_pencil_host): when KC > 1 the caller has
// made V rows [0, chunk0_w) resident in stream order on `st` and enqueued the copy of every later chunk's rows
// on a copy stream, recording ev_chunk[min(c - 1, kMaxChunkEv - 1)] after chunk c's rows, BEFORE calling
// project_launch. Chunk 0 of the projection then runs on `st`; chunks 1..KC-1 run in up to kSplitStreams
// contiguous groups, group i on s_rest[i] as soon as its rows (and their Vsum rows) are in — separate streams,
// so the groups' CTAs dispatch back to back as in one launch; the fixup counts arrivals across all launches.
// `ev_a`, `ev_b[i]` are caller-owned scratch events.
constexpr int kMaxChunkEv = 16;
constexpr int kSplitStreams = 3;
struct ProjSplit {
  cudaStream_t s_rest[kSplitStreams];
  cudaEvent_t ev_a;
  cudaEvent_t ev_b[kSplitStreams];
  const cudaEvent_t* ev_chunk;
};

ProjShape proj_shape(int m);
int project_plan(const ProjGeom& g, int sm_count, ProjPlan* pl);
// host-input pencils: a narrow chunk 0 (about a quarter of a chunk) ahead of the KC uniform chunks, so only its
// V rows are copied before the first DMMA; no change when the workspace bound leaves no room for one more chunk
void project_plan_lead(const ProjGeom& g, ProjPlan* pl);
size_t project_workspace_bytes(int d, int n, int N, int m, int sm_count);
int project_launch(const ProjGeom& g, const ProjPlan& pl, const double2* grid, const double2* U, const double2* V,
                   const double* sigma, double2* S, void* ws, int sm_count, cudaStream_t st,
                   prony_exec_info* info, cudaEvent_t wait_before_reduce = nullptr, int ell_base = 1,
                   int32_t* dev_status = nullptr, const ProjSplit* split = nullptr,
                   cudaEvent_t ev_prepped = nullptr, bool reset_status = false);
__global__ void k_combine_grid(int d, int n, int64_t box, const double2* grid, const double2* mu, double2* out);

size_t apply_workspace_bytes(int d, int n, int N);
int toeplitz_apply_launch(int d, int n, int N, const double2* grid, int ell, int conj, const double2* X, int ldx, int r,
                          double2* Yout, int ldy, void* ws, int sm_count, cudaStream_t st);

}  // namespace prony
