/*
 * iga.h — C ABI of libiga: B200-native interpolation-and-lookup formation of the
 * isogeometric linear-elasticity stiffness matrix K of a microstructured geometry
 * F∘M (Hirschler, Antolin, Buffa, arXiv 2107.09568; /root/reference/PAPER.md).
 *
 * Citations "P:L" are PAPER.md lines; "Rn" are the readings listed in DESIGN.md §4.
 *
 * Problem statement carried by the arguments:
 *   - the reference tile 𝒯^r as a multi-patch spline into [0,1]^d (Eq. 3),
 *   - the macro map ℳ = F, a single B-spline patch (Eq. 4); one tile per macro
 *     element (Eqs. 5-10),
 *   - the analysis degree p = the tile degree (the solution space recycles the tile
 *     basis, Eq. 13) and the interpolation degree q = p_π (Eq. 21),
 *   - isotropic elasticity constants E (per tile allowed) and ν.
 *
 * Pointers.  Entry points marked [any] accept host OR device pointers for their
 * array arguments (the library inspects each pointer; host arrays are staged with
 * cudaMemcpyAsync on the caller's stream).  [host] arguments must be host memory.
 * All inputs are borrowed for the duration of the call; no input is retained.
 *
 * Errors.  Nothing throws across the ABI.  Every entry point returns an iga_status;
 * on failure the outputs are unspecified and iga_last_error() (thread-local) names
 * the offending patch / tile / node.  Calls enqueue work on `stream` (a
 * cudaStream_t, NULL = legacy default stream) and synchronise that stream once at
 * the end, so that the device-side degeneracy flag can be reported.
 *
 * Concurrency.  A handle is immutable after iga_build_tables except for its
 * internal workspace (coefficients, side slots, staging buffers, profiling slots).
 * Concurrent calls on one handle — from several host threads, on the same or on
 * different streams — are safe: every entry point that uses the handle holds the
 * handle's lock until its device work is complete (each call synchronises its
 * stream before returning), so such calls are serialised, never interleaved.
 * Different handles are independent and run concurrently.
 */
#ifndef IGA_H
#define IGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IGA_OK = 0,
  IGA_EINVAL = 1,          /* invalid argument: dimension, degree, knots, sizes */
  IGA_EDEGENERATE = 2,     /* det J <= 0 at a table point (tile) or interpolation node (macro), R5 */
  IGA_ENONCONFORMING = 3,  /* tile faces / declared interfaces do not match (R10) */
  IGA_ENOMEM = 4,          /* host or device allocation failed */
  IGA_ECUDA = 5,           /* CUDA runtime error */
  IGA_ELIMIT = 6           /* problem exceeds an index-width limit of this build */
} iga_status;

/* A tensor-product B-spline patch (Eq. 2), or a NURBS patch when weights is
 * not NULL (macro map only: the rational F of the paper's torus and
 * twist, §3.3.4; tile patches must be B-splines).  [host]
 * dim: parametric = physical dimension d (2 or 3).
 * degree[k] >= 1, knots[k] (n_knots[k] values): open, non-decreasing, first = 0,
 * last = 1, interior multiplicity <= degree[k].  n_ctrl = Π_k (n_knots[k]-degree[k]-1).
 * ctrl: n_ctrl*dim doubles, point A = i0 + n0*(i1 + n1*i2) (direction-0 fastest),
 * coordinates contiguous; may be NULL where only the topology is needed (macro). */
typedef struct {
  int32_t dim;
  int32_t degree[3];
  int32_t n_knots[3];
  const double *knots[3];
  const double *ctrl;
  const double *weights;   /* n_ctrl positive weights (NURBS) or NULL (B-spline) */
} iga_spline;

/* Declared intra-tile interface (R10): face (dir_a, side_a) of patch_a is glued to
 * face (dir_b, side_b) of patch_b; side 0 = parameter 0, side 1 = parameter 1.
 * Control points on the two faces are matched by position (|Δ| <= 1e-10). */
typedef struct {
  int32_t patch_a, dir_a, side_a;
  int32_t patch_b, dir_b, side_b;
} iga_interface;

typedef struct iga_handle iga_handle;

/* Slab partition of ONE problem over n_shards processes.  The macro
 * elements are split into n_shards contiguous slabs of element layers along the slowest
 * direction (direction d-1); shard s owns the tiles of its slab and the CSR rows of the
 * nodes that first appear in it (a contiguous range of global node ids), and also forms
 * the tiles of one halo layer of the next slab so that its rows are complete.  K needs no
 * communication; iga_sensitivity returns this shard's partial gradient (its owned tiles
 * only), which the caller sums over shards (one all-reduce of n_macro_cp*d doubles).
 * NULL or n_shards = 1: the whole problem. */
typedef struct {
  int32_t n_shards;
  int32_t shard;
} iga_shard;

typedef struct {
  int32_t dim;            /* d */
  int32_t q;              /* interpolation degree p_π */
  int32_t n_pi;           /* (q+1)^d Bernstein functions N_C (Eq. 21) */
  int32_t n_k;            /* table columns κ = (i*d + j)*n_pi + C: d²·n_pi (Eq. 57) */
  int32_t k_stride;       /* padded row stride (doubles) of the table / coefficient buffers */
  int32_t n_patches;
  int32_t n_gauss;        /* Gauss points per direction per tile knot span (R3) */
  int32_t sens_path;      /* sensitivity route chosen at build: bit 0 = fused K5g (else K5x + K5a),
                             bits 8..15 = K5a split-K segments (1 = none); informational */
  int64_t n_tiles;        /* m_M = macro elements (Eq. 5), whole problem; per-tile E has this length */
  int64_t n_local_rows;   /* Σ_p n_nz,p = rows of the stacked mat𝔎 (Eqs. 56-57) */
  int64_t n_macro_cp;     /* macro control points (Eq. 4) */
  int64_t n_nodes;        /* global nodes after merging (R10), whole problem */
  int64_t n_dof;          /* n_nodes * d, interleaved DOF = node*d + a (R9): length of u, v */
  int64_t nnz;            /* scalar CSR non-zeros of the rows this handle forms (both triangles, R9) */
  int64_t n_blocks;       /* d×d structural blocks of those rows */
  int64_t n_contrib;      /* (tile, local row) -> block contributions to those rows */
  int64_t n_multi_blocks; /* blocks with more than one contribution (K4 gathers them) */
  int64_t n_side_slots;   /* contributions to those blocks (K3 side slots, d² doubles each) */
  /* shard (iga_shard; whole problem: 0, n_tiles, n_tiles, 0, n_dof) */
  int64_t tile_begin;     /* first tile of the slab (global id) */
  int64_t n_tiles_local;  /* tiles formed: slab + halo layer (local_values / coefficient rows) */
  int64_t n_tiles_owned;  /* tiles of the slab (the sensitivity's partial sum) */
  int64_t row_begin;      /* first CSR row (global scalar row = node*d + a) of this handle */
  int64_t n_rows;         /* CSR rows of this handle: row_ptr has n_rows + 1 entries */
  int32_t q_dir[3];       /* projection degree per direction (q above = the largest; unused dirs 0) */
  int32_t m_dir[3];       /* projection sample points per direction (q_dir+1: interpolation) */
  int32_t n_local_ctrl;   /* tile-local control points over all patches: the node map's row length
                             (iga_get_node_map writes n_tiles_local * n_local_ctrl values) */
} iga_sizes;

/* ---------------------------------------------------------------------------
 * iga_build_tables — offline step ("the tables are built off-line").
 *  tile_patches[n_patches]  the reference tile 𝒯^r (Eq. 3) [host]; all patches share
 *                           dim and degree (p); control points must lie in [0,1]^d.
 *  interfaces[n_interfaces] declared patch interfaces (may be NULL if 0) [host].
 *  macro_topology           degree and knots of F (ctrl ignored) [host].
 *  q                        interpolation degree (0..4).
 *  n_gauss                  Gauss points per direction per span; 0 = p + ceil((q+1)/2) (R3).
 *  shard                    NULL (whole problem) or the slab this handle forms (iga_shard).
 *  stream                   cudaStream_t used for the device work.
 *  out                      receives a new handle (owned by the caller; free with iga_free).
 * Device work: K1 (lookup tables 𝔎_p by micro Gauss quadrature, Eq. 52).
 * Host work: validation, I_coo (Eq. 56), DofMap (R10), CSR pattern + gather lists (R9).
 * Errors: EINVAL (bad spline / degrees / sizes), ENONCONFORMING (unmatched face or
 * interface control point, two points of one patch merged), EDEGENERATE (det J_T <= 0
 * at a table quadrature point), ENOMEM, ECUDA, ELIMIT (index packing limits).
 * ------------------------------------------------------------------------- */
iga_status iga_build_tables(const iga_spline *tile_patches, int32_t n_patches,
                            const iga_interface *interfaces, int32_t n_interfaces,
                            const iga_spline *macro_topology, int32_t q, int32_t n_gauss,
                            const iga_shard *shard, void *stream, iga_handle **out);

/* iga_build_tables_q — iga_build_tables with one projection degree per direction, q[k]
 * for k < d (the anisotropic spaces of §3.3.4, e.g. the twist's p_π = 3, 3, 4, P:524;
 * SURVEY §8(f) N2): n_π = Π_k (q_k+1) Bernstein functions N_C(ξ) = Π_k B_{c_k}^{q_k}(ξ_k),
 * C = c0 + (q0+1)(c1 + (q1+1)c2).  n_gauss = 0 takes R3 with the largest q_k.  Otherwise
 * identical (iga_build_tables(…, q, …) == iga_build_tables_q(…, {q, q, q}, …)). */
iga_status iga_build_tables_q(const iga_spline *tile_patches, int32_t n_patches,
                              const iga_interface *interfaces, int32_t n_interfaces,
                              const iga_spline *macro_topology, const int32_t *q, int32_t n_gauss,
                              const iga_shard *shard, void *stream, iga_handle **out);

/* iga_build_topology — host-only variant of iga_build_tables: validation, I_coo,
 * DofMap and the CSR pattern, no device work and no tables.  The handle answers
 * iga_get_sizes / iga_get_pattern (host pointers) / iga_get_block_map /
 * iga_get_node_map / iga_get_pairs; kernel entry points return IGA_EINVAL.  Lets a
 * caller size a problem (nnz, n_dof) before committing device memory. */
iga_status iga_build_topology(const iga_spline *tile_patches, int32_t n_patches,
                              const iga_interface *interfaces, int32_t n_interfaces,
                              const iga_spline *macro_topology, int32_t q, int32_t n_gauss,
                              const iga_shard *shard, iga_handle **out);
iga_status iga_build_topology_q(const iga_spline *tile_patches, int32_t n_patches,
                                const iga_interface *interfaces, int32_t n_interfaces,
                                const iga_spline *macro_topology, const int32_t *q, int32_t n_gauss,
                                const iga_shard *shard, iga_handle **out);

/* ---------------------------------------------------------------------------
 * iga_assemble — form K^π (Eq. 50) into CSR values: the hot path (§3.2.4 steps 1-4).
 *  macro_ctrl   [any] n_macro_cp*d doubles: the control net of F (Eq. 4).
 *  young        [any] E: one double (young_per_tile = 0) or n_tiles doubles (= 1).
 *  nu           Poisson ratio, -1 < ν < 0.5.
 *  csr_values   [any] nnz doubles, overwritten, ordered as the pattern of iga_get_pattern
 *               (the rows [row_begin, row_begin + n_rows) of K for a shard).  May be NULL
 *               when local_values is given: then only the non-zero components are formed
 *               (K2 + K3 into nzdata, no CSR — the paper's timing convention).
 *  local_values [any] optional (NULL = skip): n_local_rows*n_tiles_local*d² doubles receiving
 *               nzdata (Eq. 58) as local[row][t*d² + a*d + b], t = local tile index.
 * Kernels: K2 (per-tile ∇F at the (q+1)^d Gauss nodes -> Ā (Eq. 37) -> interpolation
 * coefficients, R1), K3 (FP64 DMMA contraction nzdata = mat𝔎·mat⟨Ā⟩, Eq. 58),
 * K4 (atomic-free owner-computes gather into the full symmetric CSR, R9).
 * Errors: EINVAL, EDEGENERATE (det ∇F <= 0 at an interpolation node), ECUDA.
 * ------------------------------------------------------------------------- */
iga_status iga_assemble(const iga_handle *h, const double *macro_ctrl, const double *young,
                        int32_t young_per_tile, double nu, double *csr_values,
                        double *local_values, void *stream);

/* ---------------------------------------------------------------------------
 * iga_sensitivity — g[k*d + α] = uᵀ (∂K^π/∂P_{k,α}) v for every macro control-point
 * coordinate (Eqs. 70-73; R13: u ≠ v allowed, K^π as assembled by R9).
 *  u, v  [any] n_dof doubles (interleaved DOF).   grad [any] n_macro_cp*d, overwritten
 *        (a shard: the sum over its owned tiles only; sum the shards' grads).
 * Kernels: K5a (W_t = mat𝔎ᵀ X_t, FP64 DMMA, X_t generated from u, v on the fly),
 * K5b (Ŵ = Πᵀ W, analytic reverse mode of Ā(J), chain to P), K5c (deterministic
 * reduction over the tiles sharing a control point).
 * ------------------------------------------------------------------------- */
iga_status iga_sensitivity(const iga_handle *h, const double *macro_ctrl, const double *young,
                           int32_t young_per_tile, double nu, const double *u, const double *v,
                           double *grad, void *stream);

/* ---------------------------------------------------------------------------
 * iga_volume — V^π = Σ_t t^h · d^(t) (§3.1, Eqs. 14-19): t^h the volume lookup
 * table (Eq. 18, built offline with the tables), d^(t) the projection coefficients of
 * det J_ℳ(t) (Eq. 15, with the projection of iga_set_projection).  Exact when det J_ℳ ∈ Q_q
 * (q >= d·p_M - 1, Eq. 22).  SURVEY §8(f) N3.
 *  volume [host] 1 double: the sum over this handle's (owned) tiles.
 *  grad   [any] optional n_macro_cp*d doubles: dV^π/dP (Eqs. 66-67: the adjoint field
 *         Πᵀ t^h at the projection samples times ∂det J_ℳ/∂P), owned tiles only.
 * Errors: EINVAL, EDEGENERATE, ECUDA.
 * ------------------------------------------------------------------------- */
iga_status iga_volume(const iga_handle *h, const double *macro_ctrl, double *volume, double *grad, void *stream);

/* iga_load_vector — body-force load vector for a constant body force b (Eq. 53,
 * body part): f_{node(t,A)} += b Σ_C 𝔉[A][C] d^(t)_C with the load lookup table
 * 𝔉[A][C] = ∫ R_A |det J_T| N_C∘𝒯 dθ (built offline), gathered per node in a fixed order.
 *  body_force [host] d doubles.   f [any] n_rows doubles (this handle's rows), overwritten.
 * Σ_I f_I = b·V^π.  Errors: EINVAL, EDEGENERATE, ECUDA. */
iga_status iga_load_vector(const iga_handle *h, const double *macro_ctrl, const double *body_force, double *f,
                           void *stream);

/* iga_assemble_sensitivity — iga_assemble followed by iga_sensitivity in one call (the
 * design-optimisation step: K and g together), one synchronisation at the end.  Host
 * u, v are copied on an internal stream while K is formed.  Arguments as in the two calls
 * (no local_values). */
iga_status iga_assemble_sensitivity(const iga_handle *h, const double *macro_ctrl, const double *young,
                                    int32_t young_per_tile, double nu, const double *u, const double *v,
                                    double *csr_values, double *grad, void *stream);

/* ---------------------------------------------------------------------------
 * iga_apply — matrix-free y = K^π u (Eq. 74: "the multiplication of a vector
 * with the system matrix with only the lookup table and the projection coefficients at
 * hand").  K is never stored: K2, then the K3 contraction whose epilogue
 * multiplies every element block with u and sums the products of each run of equal local
 * row / column index into a partial slot, then a gather of the partials per node in a
 * fixed order (deterministic, no atomics).  Equals the CSR product of iga_assemble's K.
 *  u  [any] n_dof doubles (global).   y [any] n_rows doubles (this handle's rows), overwritten.
 * Device memory: n_tiles_local * P * d doubles of partials, allocated by the first call.
 * Errors: EINVAL, EDEGENERATE, ENOMEM, ECUDA.
 * ------------------------------------------------------------------------- */
iga_status iga_apply(const iga_handle *h, const double *macro_ctrl, const double *young,
                     int32_t young_per_tile, double nu, const double *u, double *y, void *stream);

/* iga_interpolate — K2 only (parity): coefficients ⟨Ā_ij⟩_C of every tile, written as
 * coef[(t*d² + a*d + b)*k_stride + κ] with κ = (i*d + j)*n_pi + C.  [any] pointers. */
iga_status iga_interpolate(const iga_handle *h, const double *macro_ctrl, const double *young,
                           int32_t young_per_tile, double nu, double *coef, void *stream);

/* iga_set_projection — the projection Π^H of the macro field (Eq. 20) onto Q_q: the L2
 * projection of Eqs. 23-24 (and 42) with its mass matrix and right-hand side integrated
 * by an m-point Gauss rule per direction, m >= q_k+1 for every k.
 * m = 0 (or m = q+1 for isotropic q, the default) is interpolation at the q_k+1 Gauss
 * nodes of each direction (reading R1, equal to that projection); larger m converge to the
 * exact L2 projection (exact once 2m-1 >= q + the degree of Ā's polynomial part).  Applies
 * to iga_assemble / iga_sensitivity / iga_interpolate / iga_apply / iga_volume /
 * iga_load_vector; the tables do not depend on m.  iga_get_projection returns m as set
 * (q+1 for isotropic interpolation, 0 for anisotropic interpolation).
 * Errors: EINVAL (0 < m < q_k+1 or m > 8), ELIMIT (per-tile staging exceeds shared
 * memory, e.g. m > 5 in 3D). */
iga_status iga_set_projection(iga_handle *h, int32_t m);
iga_status iga_get_projection(const iga_handle *h, int32_t *m);

/* ---------------------------------------------------------------------------
 * iga_projection_error — the a-priori projection error of Eq. 59, evaluated "by a
 * simple sampling-based approach ... a priori to the assembly":
 *   e_t = max_{ξ ∈ S} ‖Ā^(t)(ξ) − Π^H Ā^(t)(ξ)‖_F / ‖Ā^(t)(ξ)‖_F,   E_proj = max_t e_t,
 * ‖·‖_F over all d⁴ components, S = n_samples equispaced points per direction of the
 * element-local cube, endpoints included (reading R18); Ā ∝ E, so E does not enter.
 * No tables are needed: this is the a-priori step of the degree selection.
 *  macro      the macro map F with control points (and weights for NURBS) [host].
 *  q          d projection degrees (0..4).   m_extra >= 0: q_k+1+m_extra Gauss points per
 *             direction (0 = interpolation, R1; else the L2 projection of Eqs. 23-24).
 *  nu         Poisson ratio.   n_samples in [2, 8] (0 = 8).
 *  e_max      [host] E_proj.   e_tile [any] optional n_tiles doubles: e_t per tile.
 * Device work: one CTA per tile (K2's passes, then evaluation passes at S); fixed order,
 * exact max.  Errors: EINVAL, EDEGENERATE (det ∇F <= 0 at a node or sample), ELIMIT
 * (staging exceeds shared memory), ENOMEM, ECUDA. */
iga_status iga_projection_error(const iga_spline *macro, const int32_t *q, int32_t m_extra, double nu,
                                int32_t n_samples, double *e_max, double *e_tile, void *stream);

/* iga_select_degree — Eq. 65: find p_π with E_proj(p_π) <= tol, starting from
 * the macro map's degrees and enriching or coarsening the space.  Reading
 * R19: uniformly, q(s) = (max(p_M,k + s, 0))_k; returns the smallest such q(s) (for the
 * twist's macro degrees 1, 1, 2 this gives 3, 3, 4 at s = 2).
 *  tol > 0;  m_extra, n_samples as in iga_projection_error;  q_max: largest admissible
 *  degree (<= 0: 4).   q_out [host] d degrees;  e_out [host, optional] E_proj(q_out).
 * Errors: ELIMIT if no q(s) with max_k q_k <= q_max meets tol (q_out, e_out then hold the
 * largest one tried); otherwise as iga_projection_error. */
iga_status iga_select_degree(const iga_spline *macro, double nu, double tol, int32_t m_extra, int32_t n_samples,
                             int32_t q_max, int32_t *q_out, double *e_out, void *stream);

/* Accessors.  iga_get_sizes: [host] out. */
iga_status iga_get_sizes(const iga_handle *h, iga_sizes *out);

/* iga_get_pattern — row_ptr (n_rows+1 int64, starting at 0), col_idx (nnz int32, global
 * columns); either may be NULL.  [any] pointers. */
iga_status iga_get_pattern(const iga_handle *h, int64_t *row_ptr, int32_t *col_idx);

/* iga_get_block_map — for local tiles [t_begin, t_end): (pos(I*d,J*d), pos(J*d,I*d)) per
 * (tile, local row) as 2 int64 each, tile-major (R9); -1 where the row is not this
 * handle's. [host] out. */
iga_status iga_get_block_map(const iga_handle *h, int64_t t_begin, int64_t t_end, int64_t *out);

/* iga_get_node_map — global node[t*n_local_ctrl + off_p + A] for the local tiles (R10).
 * [host] out (n_tiles_local * Σ_p n_ctrl,p int32).  */
iga_status iga_get_node_map(const iga_handle *h, int32_t *out);

/* iga_get_tables — the stacked table mat𝔎 (n_local_rows × n_k, row-major, unpadded). [any] */
iga_status iga_get_tables(const iga_handle *h, double *out);

/* iga_get_pairs — (A, B) of every stacked table row, 2 int32 per row. [host] */
iga_status iga_get_pairs(const iga_handle *h, int32_t *out);

/* Per-kernel device time accumulated by iga_assemble / iga_sensitivity calls while
 * profiling is enabled (CUDA events on the caller's stream).  IGA_N_PROF slots:
 * 0 K2 interpolate, 1 K3 contraction + fused scatter, 2 K4 multi-contribution gather,
 * 3 K5a W-GEMM, 4 K5b reverse, 5 K5c reduce, 6 host<->device staging, 7 K5x X generation,
 * 8 K3 nzdata output (local_values), 9 matrix-free apply (K3 apply epilogue + gather).
 * enable != 0 resets the accumulators. */
#define IGA_N_PROF 10
iga_status iga_set_profiling(iga_handle *h, int32_t enable);
iga_status iga_get_kernel_times(const iga_handle *h, double *ms_out /* IGA_N_PROF */,
                                int64_t *launches_out /* IGA_N_PROF */);

void iga_free(iga_handle *h);
const char *iga_last_error(void);
const char *iga_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IGA_H */
