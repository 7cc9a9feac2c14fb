// vandermonde_ls.cuh — host/device interface of the Vandermonde / LS kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace prony {

constexpr int kMaxM = PRONY_MAX_M;
#ifndef PRONY_VLS_TILE
#define PRONY_VLS_TILE 16
#endif
constexpr int kTile = PRONY_VLS_TILE;  // columns of A per smem tile of k_vls
constexpr int kVlsThreads = 512;   // 16 warps (DMMA warp engine)
constexpr int kSolveThreads = 512;

constexpr int kVlsMaxUnits = 32;  // lower-triangle warp units (m <= 128 needs 20 at 4 n-tiles each)

struct VlsParams {
  int d, n, m, CB, cap, nunits;
  int unit[kVlsMaxUnits][3];  // (m-tile, first n-tile, n-tiles) per warp unit
  int64_t col_begin, col_end;
  const double2* pw;
  const double2* grid;
  double2* A;
  double2* Gpart;
  double2* bpart;
};

size_t ls_workspace_bytes(int d, int n, int m, int sm_count);
int ls_launch(int d, int n, int m, int N, const double2* z, const double2* grid, int64_t col_begin, int64_t col_end,
              double2* A, double2* G, double2* b, double2* c, double* t, void* ws, int32_t* status, int sm_count,
              cudaStream_t st, prony_exec_info* info);

int ls_solve_launch(int d, int m, const double2* G, const double2* b, const double2* z, double2* c, double* t,
                    void* ws, int32_t* status, cudaStream_t st);

}  // namespace prony
