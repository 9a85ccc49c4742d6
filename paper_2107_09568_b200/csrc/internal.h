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
#define IGA_MAXM 8          // max L2-projection points per direction (NEXT N2)
#define IGA_KCHUNK 16       // GEMM k-chunk; k_stride is a multiple of it
#ifndef IGA_K3_BM
#define IGA_K3_BM 64        // K3 CTA rows (table rows): 4 MMA warps, 4 CTAs per SM
#endif
#ifndef IGA_K3_CL
#ifdef IGA_EXPERIMENT_K3_CLUSTER
#define IGA_K3_CL 8         // K3 CTAs per thread-block cluster (transposed scatter pass pooled over the cluster)
#else
#define IGA_K3_CL 1
#endif
#endif
#define IGA_K5_BM 256       // K5a CTA rows (κ): 16 MMA warps, all κ rows of a 3D q = 2 problem in one CTA
#define IGA_GEMM_BN 72      // K3/K5a CTA columns (tiles × d²): 8 tiles in 3D, 18 in 2D

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

// one d×d block of K that several (tile, local row) contributions share (K4 gather)
struct MultiBlock {
  int64_t off_ij;      // scalar CSR offset of element (0,0) of block (I,J)
  int64_t off_ji;      // ... of block (J,I)
  int32_t stride_i;    // d * (blocks in block row I) = scalar row pitch of row I
  int32_t stride_j;
};

// K4 pass descriptor (one per multi block and pass, in the pass's store order): where the
// pass writes (off < 0: nothing, i.e. a diagonal block in pass 2 or a row of another shard),
// the row pitch, the block's slot range and whether the block is diagonal (upper triangle
// mirrored) — one 16-B load instead of the mperm → mblk / mslot0 chain.
// sn = stride | ns << 17 | diag << 31 (stride = d·blocks of the row < 3·32768 < 2^17).
constexpr int K4_MAX_NS = 1 << 14;
struct __align__(16) K4Desc {
  int64_t off;
  int32_t s0;       // first side slot (even: the block's slots start 16-B aligned)
  uint32_t sn;
};
inline K4Desc k4_desc(int64_t off, int32_t stride, int32_t s0, int32_t ns, bool diag) {
  return K4Desc{off, s0, (uint32_t)stride | ((uint32_t)ns << 17) | (diag ? 1u << 31 : 0u)};
}

struct Handle {
  int d = 0, p = 0, q = 0, n_g = 0, npi = 0, nk = 0, kstride = 0;
  int qv[3] = {0, 0, 0};         // per-direction projection degrees (anisotropic Q); q = max
  bool iso = true;               // all qv equal and (after set_projection) all mv equal
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
  std::vector<double> mweights;  // NURBS macro weights (empty: B-spline)
  std::vector<int> mel_span[3];
  int64_t n_cp = 0;
  // tiles: global count; this handle's local tiles [t_base, t_base + n_tiles) of which the
  // first n_tiles_own are owned (the rest is the halo layer of a shard)
  int64_t n_tiles_glob = 0, t_base = 0, n_tiles = 0, n_tiles_own = 0;
  int32_t n_shards = 1, shard = 0;
  // global numbering / pattern
  // nodes: global count; owned (CSR) rows are nodes [node_base, node_base + n_nodes);
  // n_dof = global DOF count (length of u, v); nnz / n_blocks are the owned rows'
  int64_t n_nodes_glob = 0, node_base = 0, n_nodes = 0, n_dof = 0, nnz = 0, n_blocks = 0, n_contrib = 0;
  std::vector<int32_t> node_map;     // [n_tiles][n_local_ctrl]
  std::vector<int64_t> brow_ptr;     // [n_nodes+1]
  std::vector<int32_t> bcol;         // [n_blocks]
  // K3 fused-epilogue maps (reading R9; until upload)
  std::vector<int64_t> rowinfo;      // [n_tiles*n_local_ctrl] (brow_ptr[I] << 24) | blocks in row I
  std::vector<int32_t> emap;         // [n_tiles*M] >= 0: rank(J in row I) | rank(I in row J) << 16; < 0: -(slot+1)
  int64_t n_multi = 0, n_slots = 0;  // blocks with > 1 contribution, and their contributions
  int64_t n_slot_cap = 0;             // side slots allocated (per block: n contributions rounded up to even)
  std::vector<MultiBlock> mblk;      // [n_multi]
  std::vector<int32_t> mslot0;       // [n_multi+1] first slot of each multi block
  std::vector<int32_t> mperm;        // [n_multi] multi blocks in (J, I) order (K4 transposed pass)
  std::vector<uint8_t> slot_tr;      // [n_slots] 1 = slot holds the (J,I)-oriented block
  std::vector<K4Desc> k4d;           // [2][n_multi] pass 1 in (I,J) order, pass 2 in (J,I) order
  // operand layouts (fragment-major, device_common.cuh fm_index)
  int64_t Mpad = 0;                  // rows of d_tabA (multiple of IGA_K3_BM · IGA_K3_CL)
  int64_t Npad = 0;                  // rows of d_coef / d_X (IGA_GEMM_BN per block of tpc tiles)
  int64_t k5_rows = 0;               // κ rows of d_tabAT (multiple of IGA_K5_BM)
  // Eq. 38-reduced contraction (device_common.cuh sym_index): the GEMM
  // columns are part 1 = P1 pairs × n_π (T_ii, T_ij + T_ji) against the symmetric outputs
  // and part 2 = P2 pairs × n_π (T_ij − T_ji) against the antisymmetric ones; an N-block
  // holds tpc tiles, block column n = o*tpc + tl (o < n_p1: symmetric output o, else the
  // antisymmetric output o - n_p1)
  int n_p1 = 0, n_p2 = 0;            // d(d+1)/2, d(d-1)/2
  int tpc = 8;                       // tiles per N-block: 8 (3D), 16 (2D)
  int ks3 = 0;                       // K3 k stride of d_tabA / d_coef (multiple of 16)
  int k3_split = 0, k3_steps = 0;    // K3 k-step where part 2 starts; k-steps (parts padded to 4)
  int k5_split = 0, k5_kap = 0;      // K5a κ row where part 2 starts; rows used (parts padded to 8)
  // K5a balance: logical 8-row κ group g -> physical group (block·16 + warp·2 + mi), chosen so
  // that every CTA and sub-partition carries a similar DMMA load (part-1 groups cost 6 column
  // tiles, part-2 groups 3); per (κ-block, warp) the parts of its two groups (mode p0·3 + p1)
  int k5_nseg = 1;                   // K5a split-K segments (small problems: fill the SMs)
  double *d_Wpart = nullptr;         // [k5_nseg][blocks·72][k5_rows] partial Y (k5_nseg > 1)
  std::vector<int32_t> k5_gphys;
  std::vector<uint8_t> k5_mode;
  // K5g column split (3D): per (κ-block, warp) an extra single-column piece (local 8-row
  // group | column tile << 16, or -1) that evens the sub-partition DMMA loads (modes 9-12)
  std::vector<int32_t> k5_extra;
  int32_t *d_k5_gphys = nullptr;
  uint8_t *d_k5_mode = nullptr;
  int32_t *d_k5_extra = nullptr;
  int64_t Kp = 0;                    // K5a reduction length: table rows, each patch padded to 16
  int max_patch_ctrl = 0;
  std::vector<int32_t> pcol;         // [n_patches+1] first padded column of each patch
  std::vector<int32_t> k5_pair;      // [Kp] patch-local (A | B << 16), -1 = padding
  std::vector<int32_t> k5_col;       // [M] padded column of each table row
  std::vector<uint8_t> tperm;        // [Mpad] K3 transposed-pass row order within each 64-row block
  std::vector<uint16_t> cperm;       // [Mpad] the same order within each IGA_K3_CL·64-row cluster block
  std::vector<int4> rowdesc;         // [Mpad] (see d_rowdesc)
  // matrix-free apply (NEXT N1, Eq. 74): per 128-row block, runs of rows with equal A (row
  // order) and equal B (tperm order) are summed into one partial slot each (tile-independent)
  int64_t P = 0;                     // partial slots per tile
  std::vector<uint16_t> g1len, g2len;   // [Mpad] run length (<= 64) | position in the run << 8; 0 for dead rows
  std::vector<int32_t> g1slot, g2slot;  // [Mpad] slot of that run
  std::vector<int32_t> sA_ptr, sA_slot; // [nl+1], [P]: slots whose key is local control point A
  std::vector<int64_t> inv_ptr;      // [n_nodes+1] owned node -> its (tile, A) occurrences
  std::vector<int32_t> inv_ent;      // lt*nl + A, sorted
  bool on_device = false;
  // projection operator (Eqs. 23-24 with an m_k-point Gauss rule in direction k; m_k = q_k+1:
  // interpolation at the Gauss nodes, reading R1): coef_c = Σ_i Pi1[k][c*m_k + i] f(x_i)
  int m_proj = 0;                // as requested: q+1 (isotropic interpolation), 0 (anisotropic interpolation) or m
  int mv[3] = {1, 1, 1};
  int ns = 1;                    // Π_k m_k sample nodes per tile
  double interp_x[3][IGA_MAXM];
  double Pi1[3][(IGA_MAXQ + 1) * IGA_MAXM];
  // device buffers
  double *d_table = nullptr;     // [M][kstride] row-major (K1 output, accessor)
  double *d_tabA = nullptr;      // FM [Mpad][ks3], BR = IGA_K3_BM (K3 A operand, sym columns)
  double *d_tabAT = nullptr;     // FM [k5_rows][Kp], BR = IGA_K5_BM (K5a A operand, sym rows)
  double *d_coef = nullptr;      // FM [Npad][ks3], BR = IGA_GEMM_BN (K3 B operand, sym coefficients)
  double *d_side = nullptr;      // [n_slots][d*d] multi-contribution blocks (K3 -> K4)
  double *d_W = nullptr;         // [Npad][k5_rows] K5a output Y (block column order, sym κ rows)
  double *d_X = nullptr;         // FM [Npad][Kp], BR = IGA_GEMM_BN (K5a B operand, from u, v)
  double *d_gpart = nullptr;     // [n_tiles][n_el_cp][d]
  int32_t *d_node_map = nullptr;
  int32_t *d_pairA = nullptr, *d_pairB = nullptr;
  int64_t *d_row_ptr = nullptr;
  int32_t *d_col_idx = nullptr;
  int64_t *d_brow_ptr = nullptr;
  int32_t *d_bcol = nullptr;
  int64_t *d_rowinfo = nullptr;
  int32_t *d_emap = nullptr;
  MultiBlock *d_mblk = nullptr;   // (not uploaded: K4 reads d_k4d)
  K4Desc *d_k4d = nullptr;
  int32_t *d_mslot0 = nullptr;
  int32_t *d_mperm = nullptr;
  uint8_t *d_slot_tr = nullptr;
  int32_t *d_k5_pair = nullptr;
  int32_t *d_k5_col = nullptr;   // [M]
  uint8_t *d_tperm = nullptr;    // [Mpad]
  uint16_t *d_cperm = nullptr;   // [Mpad]
  int4 *d_rowdesc = nullptr;     // [Mpad] K3p store warps: {A | B << 16, At | Bt << 16, tperm, 0} (A = -1: padding)
  uint16_t *d_g1len = nullptr, *d_g2len = nullptr;
  int32_t *d_g1slot = nullptr, *d_g2slot = nullptr, *d_sA_ptr = nullptr, *d_sA_slot = nullptr, *d_inv_ent = nullptr;
  int64_t *d_inv_ptr = nullptr;
  double *d_part = nullptr;      // [n_tiles][P][d] apply partials (allocated by the first iga_apply)
  double *d_ug = nullptr;        // [n_tiles][n_local_ctrl][d] u gathered per tile (iga_apply)
  // volume / load (NEXT N3)
  double *d_F = nullptr;         // [n_local_ctrl][npi] load table 𝔉 (Eq. 53)
  double *d_th = nullptr;        // [npi] volume table t^h (Eq. 18)
  double *d_det = nullptr;       // [n_tiles][npi] projection coefficients of det J_ℳ (Eq. 15)
  double *d_Vt = nullptr;        // [n_tiles] tile volumes, [n_tiles] + 1: the total
  int32_t *d_patch_info = nullptr; // [n_patches][3]: first K5a chunk, ctrl_off, n_ctrl (+ sentinel chunk)
  double *d_mknots = nullptr;    // macro knots, 3 directions concatenated
  double *d_mweights = nullptr;  // [n_cp] NURBS macro weights (nullptr: B-spline)
  int32_t *d_mspan = nullptr;    // element -> knot span, 3 directions concatenated
  int *d_flag = nullptr;         // [0] error flag, [1] tile, [2] node, [3] K3p tile counter
  // staging (host pointers in [any] arguments)
  static constexpr int N_STAGE = 6;
  cudaStream_t aux_stream = nullptr;   // iga_assemble_sensitivity: u, v copies beside K formation
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double *d_stage[N_STAGE] = {nullptr};   // grow-only device copies of host [any] arguments
  size_t stage_cap[N_STAGE] = {0};
  // profiling
  bool profiling = false;
  double prof_ms[IGA_N_PROF] = {0};
  int64_t prof_launches[IGA_N_PROF] = {0};
  std::vector<cudaEvent_t> ev_pool;
  ~Handle();
};

// --- device constants shared by kernels (set by api) ---
struct InterpConst {
  int d, q, pm[3], mn[3], mel[3], moff[3], soff[3];   // offsets of direction k in d_mknots / d_mspan
  int64_t t_base;        // global id of local tile 0
  const double *mweights;   // NURBS macro weights (nullptr: B-spline)
  int64_t n_own;         // owned local tiles (sensitivity reduction)
  int m;                 // isotropic case: projection points per direction (q+1: interpolation)
  int qv[3], mv[3];      // per-direction degrees and sample points (directions >= d: 0 and 1)
  int npi, ns, iso;      // Π (q_k+1), Π m_k, all directions equal
  double Pi1[3][(IGA_MAXQ + 1) * IGA_MAXM];   // [k][(q_k+1) x m_k]
  double x[3][IGA_MAXM];
};

// --- kernel launchers (kernels_*.cu) ---
cudaError_t launch_tables(const Handle &h, const DevPatch *dpatches, int n_patches,
                          const double *d_tile_ctrl, const double *d_tile_knots, const int *d_tile_elspan,
                          const double *d_gx, const double *d_gw, int total_pts, cudaStream_t s);
// fm = true: FM layout into d_coef-shaped buffer; false: row-major coef[n][kstride]
cudaError_t launch_interpolate(const Handle &h, const double *ctrl, const double *young, int young_per_tile,
                               double nu, double *coef, bool fm, cudaStream_t s);
cudaError_t launch_pack_tables(const Handle &h, cudaStream_t s);
// K3: vals != nullptr -> fused CSR epilogue (+ side slots); local != nullptr -> local[M][N] output
cudaError_t launch_contraction(const Handle &h, double *vals, double *local, cudaStream_t s);
cudaError_t launch_scatter_multi(const Handle &h, double *vals, cudaStream_t s);
cudaError_t launch_apply(const Handle &h, const double *u, double *y, cudaStream_t s);   // K3 apply + gather
cudaError_t launch_expand_pattern(const Handle &h, cudaStream_t s);
cudaError_t launch_sens_X(const Handle &h, const double *u, const double *v, cudaStream_t s);
cudaError_t launch_sens_W(const Handle &h, double *W, cudaStream_t s);
// K5x fused into K5a (cudaErrorNotSupported: staging does not fit, run K5x + K5a)
cudaError_t launch_sens_XW(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s);
bool sens_xw_fits(const Handle &h);
size_t k5x_smem_bytes(int d, int max_patch_ctrl);
cudaError_t launch_sens_reverse(const Handle &h, const double *ctrl, const double *young, int young_per_tile,
                                double nu, const double *W, double *gpart, cudaStream_t s);
cudaError_t launch_sens_reduce(const Handle &h, const double *gpart, double *grad, cudaStream_t s);
cudaError_t launch_volume(const Handle &h, const double *ctrl, double *d_volume, double *gpart, cudaStream_t s);
cudaError_t launch_load(const Handle &h, const double *b, double *f, cudaStream_t s);
InterpConst make_interp_const(const Handle &h);

// host build steps (host_build.cpp)
iga_status build_host(Handle &h, const iga_spline *tile, int n_patches, const iga_interface *ifc,
                      int n_ifc, const iga_spline *macro, const int *q, int n_gauss, const iga_shard *shard);
iga_status parse_macro(Handle &h, const iga_spline *macro, int d);   // macro knots / elements / weights
iga_status set_degrees(Handle &h, const int *q);                      // qv, q, iso, npi, nk, kstride
void gauss_legendre01(int n, double *x, double *w);
// host: Pi1, x per direction; m = 0: interpolation (m_k = q_k+1), else m_k = m for every k
iga_status set_projection(Handle &h, int m);
iga_status set_projection_v(Handle &h, const int *mv);
size_t macro_smem_bytes(int d, int ns);
size_t k5b_smem_bytes(const Handle &h, int ns);
// a-priori projection error (Eq. 59) per tile of the macro map in h (device work)
cudaError_t launch_projection_error(const Handle &h, const double *ctrl, double nu, int n_s, double *e_tile,
                                    cudaStream_t s);
size_t projection_error_smem_bytes(int d, int ns, int n_s, int npi);
iga_status upload_topology(Handle &h);

}  // namespace iga
