// internal.h — libiga internals shared by the host builder and the CUDA kernels.
// Not part of the ABI (see include/iga.h).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/iga.h"

#define IGA_MAXD 3
#define IGA_MAXP 4          // max spline degree (tile and macro)
#define IGA_MAXQ 4          // max interpolation degree
#define IGA_KCHUNK 16       // GEMM k-chunk; k_stride is a multiple of it

namespace iga {

void set_error(const char *fmt, ...);

struct PatchInfo {
  int deg[3];
  int n[3];            // control points per direction
  int n_ctrl;
  int ctrl_off;        // offset of this patch's points in the tile-local numbering
  int n_span[3];       // elements per direction
  int span_off;        // offset of this patch's spans in the global span list
  int n_spans;         // Π n_span
  int pt_off;          // offset of this patch's quadrature points
  int n_nz;            // |I_coo|
  int row_off;         // offset in the stacked table rows
  std::vector<double> knots[3];
  std::vector<int> el_span[3];   // knot-span index of element e
  std::vector<double> ctrl;      // n_ctrl * d
};

// device-side description of one tile patch (for K1)
struct DevPatch {
  int deg;             // common tile degree p
  int n[3];
  int n_span[3];
  int ctrl_off;        // into d_tile_ctrl (points)
  int knot_off[3];     // into d_tile_knots
  int elspan_off[3];   // into d_tile_elspan
  int pt_off;          // first quadrature point of the patch
  int n_spans;
};

struct Handle {
  int d = 0, p = 0, q = 0, n_g = 0, npi = 0, nk = 0, kstride = 0;
  int n_patches = 0;
  std::vector<PatchInfo> patches;
  int n_local_ctrl = 0;
  int64_t M = 0;                 // stacked table rows
  std::vector<int32_t> pairA, pairB;   // tile-local ctrl index (incl. patch offset) per row
  // macro topology
  int pm[3] = {0, 0, 0};
  int mn[3] = {1, 1, 1};         // macro control points per dir
  int mel[3] = {1, 1, 1};        // macro elements per dir
  std::vector<double> mknots[3];
  std::vector<int> mel_span[3];
  int64_t n_cp = 0, n_tiles = 0;
  // global numbering / pattern
  int64_t n_nodes = 0, n_dof = 0, nnz = 0, n_blocks = 0, n_contrib = 0;
  int row_bits = 0;
  std::vector<int32_t> node_map;     // [n_tiles][n_local_ctrl]
  std::vector<int64_t> brow_ptr;     // [n_nodes+1]
  std::vector<int32_t> bcol;         // [n_blocks]
  std::vector<uint8_t> bcnt;         // [n_blocks] contributions per block (until upload)
  std::vector<uint32_t> contrib;     // packed gather list (until upload)
  std::vector<int64_t> cstart;       // [n_nodes+1] (until upload)
  bool on_device = false;
  // interpolation operator
  double interp_x[IGA_MAXQ + 1];
  double Pi1[(IGA_MAXQ + 1) * (IGA_MAXQ + 1)];   // V1^{-1}
  // device buffers
  double *d_table = nullptr;     // [M][kstride]
  double *d_tableT = nullptr;    // [kstride][M] (K5a A-operand)
  double *d_coef = nullptr;      // [n_tiles*d*d][kstride]
  double *d_local = nullptr;     // [M][N], N = n_tiles*d*d
  double *d_W = nullptr;         // [N][kstride]
  double *d_gpart = nullptr;     // [n_tiles][n_el_cp][d]
  int32_t *d_node_map = nullptr;
  int32_t *d_pairA = nullptr, *d_pairB = nullptr;
  int64_t *d_row_ptr = nullptr;
  int32_t *d_col_idx = nullptr;
  int64_t *d_brow_ptr = nullptr;
  int32_t *d_bcol = nullptr;
  uint8_t *d_bcnt = nullptr;
  int64_t *d_cstart = nullptr;   // [n_nodes+1] start of each node's contributor list
  uint32_t *d_contrib = nullptr; // packed (t, row, transposed)
  double *d_mknots = nullptr;    // macro knots, 3 directions concatenated
  int32_t *d_mspan = nullptr;    // element -> knot span, 3 directions concatenated
  int *d_flag = nullptr;         // [0] error flag, [1] tile, [2] node
  // staging (host pointers in [any] arguments)
  double *d_stage_ctrl = nullptr, *d_stage_young = nullptr, *d_stage_u = nullptr, *d_stage_v = nullptr;
  double *d_stage_out = nullptr; size_t stage_out_bytes = 0;
  // profiling
  bool profiling = false;
  double prof_ms[8] = {0};
  int64_t prof_launches[8] = {0};
  std::vector<cudaEvent_t> ev_pool;
  ~Handle();
};

// --- device constants shared by kernels (set by api) ---
struct InterpConst {
  int d, q, pm[3], mn[3], mel[3], moff[3], soff[3];   // offsets of direction k in d_mknots / d_mspan
  double Pi1[(IGA_MAXQ + 1) * (IGA_MAXQ + 1)];
  double x[IGA_MAXQ + 1];
};

// --- kernel launchers (kernels_*.cu) ---
cudaError_t launch_tables(const Handle &h, const DevPatch *dpatches, int n_patches,
                          const double *d_tile_ctrl, const double *d_tile_knots, const int *d_tile_elspan,
                          const double *d_gx, const double *d_gw, int total_pts, cudaStream_t s);
cudaError_t launch_interpolate(const Handle &h, const double *ctrl, const double *young, int young_per_tile,
                               double nu, double *coef, cudaStream_t s);
cudaError_t launch_contraction(const Handle &h, const double *A, const double *B, double *C,
                               int64_t M, int64_t N, int K, int kstride, cudaStream_t s);
cudaError_t launch_scatter(const Handle &h, const double *local, double *vals, cudaStream_t s);
cudaError_t launch_expand_pattern(const Handle &h, cudaStream_t s);
cudaError_t launch_sens_W(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s);
cudaError_t launch_sens_reverse(const Handle &h, const double *ctrl, const double *young, int young_per_tile,
                                double nu, const double *W, double *gpart, cudaStream_t s);
cudaError_t launch_sens_reduce(const Handle &h, const double *gpart, double *grad, cudaStream_t s);
InterpConst make_interp_const(const Handle &h);

// host build steps (host_build.cpp)
iga_status build_host(Handle &h, const iga_spline *tile, int n_patches, const iga_interface *ifc,
                      int n_ifc, const iga_spline *macro, int q, int n_gauss);
void gauss_legendre01(int n, double *x, double *w);
iga_status upload_topology(Handle &h);

}  // namespace iga
