// kernels_macro.cu — macro-scale kernels.
//
// K2 (interpolation, Eq. 42 in interpolation form, reading R1): per tile,
//   ∇F at the (q+1)^d tensor Gauss nodes of the element-local cube (Eq. 7 frame, R4),
//   Ā_ij[a,b] = D (λ ǧ_i[a] ǧ_j[b] + μ ǧ_j[a] ǧ_i[b] + μ (ǧ_i·ǧ_j) δ_ab)   (Eq. 37, App. A)
//   and the coefficients ⟨Ā⟩ = (V1⁻¹)^{⊗d} · samples (sum-factorised, one pass per direction).
//   For K3 it writes the 45 (3D) / 10 (2D) distinct symmetric / antisymmetric halves
//   ½(⟨Ā_ij[a,b]⟩ ± ⟨Ā_ij[b,a]⟩) of the Eq. 38-reduced contraction; for
//   iga_interpolate all d⁴ components.  The only large traffic is the coefficient write.
//
// K5b (sensitivity, Eqs. 70-72): Ŵ_t = Πᵀ W_t, then at each node the analytic
//   reverse mode of S = ⟨Ŵ, Ā(J)⟩:
//     ∂S/∂J = S Gᵀ - Gᵀ Q Gᵀ,  G = J⁻¹,  Q = D(λ ∂T1/∂G + μ ∂T2/∂G + μ ∂T3/∂G)
//   chained to the macro control points through ∂J/∂P = h_β ∂_β N_k.
// K5c: deterministic reduction of the per-tile partials over the tiles sharing a
//   control point (fixed tile order, no atomics).
#include <algorithm>
#include <cmath>
#include "device_common.cuh"

namespace iga {

InterpConst make_interp_const(const Handle &h) {
  InterpConst ic;
  ic.d = h.d;
  ic.q = h.q;
  int off = 0, soff = 0;
  for (int k = 0; k < 3; ++k) {
    ic.pm[k] = h.pm[k];
    ic.mn[k] = h.mn[k];
    ic.mel[k] = h.mel[k];
    ic.moff[k] = off;
    ic.soff[k] = soff;
    off += (k < h.d) ? (int)h.mknots[k].size() : 0;
    soff += (k < h.d) ? (int)h.mel_span[k].size() : 0;
  }
  ic.t_base = h.t_base;
  ic.mweights = h.d_mweights;
  ic.n_own = h.n_tiles_own;
  ic.m = h.mv[0];
  ic.npi = h.npi;
  ic.ns = h.ns;
  ic.iso = h.iso ? 1 : 0;
  for (int k = 0; k < 3; ++k) {
    ic.qv[k] = h.qv[k];
    ic.mv[k] = h.mv[k];
    for (int i = 0; i < (IGA_MAXQ + 1) * IGA_MAXM; ++i) ic.Pi1[k][i] = h.Pi1[k][i];
    for (int i = 0; i < IGA_MAXM; ++i) ic.x[k][i] = h.interp_x[k][i];
  }
  return ic;
}

// Shared per-tile macro data: 1D basis at the nodes and the active control points.
template <int D>
struct MacroTile {
  double B1[D][IGA_MAXM][IGA_MAXP + 1];
  double D1[D][IGA_MAXM][IGA_MAXP + 1];   // derivative w.r.t. ξ_k (includes span length)
  double P[(D == 2 ? (IGA_MAXP + 1) * (IGA_MAXP + 1) : (IGA_MAXP + 1) * (IGA_MAXP + 1) * (IGA_MAXP + 1)) * D];
  double Wt[D == 2 ? (IGA_MAXP + 1) * (IGA_MAXP + 1) : (IGA_MAXP + 1) * (IGA_MAXP + 1) * (IGA_MAXP + 1)];   // NURBS weights
  int nact;
  int rational;
};

template <int D>
__device__ void load_macro_tile(const InterpConst &c_ip, MacroTile<D> &mt, int64_t t, const double *__restrict__ ctrl,
                                const double *__restrict__ mknots, const int *__restrict__ mspan,
                                int tid = threadIdx.x, int nthr = blockDim.x) {
  int e[3] = {0, 0, 0};
  int64_t tmp = t;
  for (int k = 0; k < D; ++k) { e[k] = (int)(tmp % c_ip.mel[k]); tmp /= c_ip.mel[k]; }
  for (int idx = tid; idx < D * IGA_MAXM; idx += nthr) {   // sample point m of direction k
    const int k = idx / IGA_MAXM, m = idx % IGA_MAXM;
    if (m >= c_ip.mv[k]) continue;
    const double *U = mknots + c_ip.moff[k];
    int s = mspan[c_ip.soff[k] + e[k]];
    double h = U[s + 1] - U[s];
    double N[IGA_MAXP + 1], dN[IGA_MAXP + 1];
    bspline_eval_reg(U, c_ip.pm[k], s, U[s] + h * c_ip.x[k][m], N, dN);
    for (int r = 0; r <= c_ip.pm[k]; ++r) {
      mt.B1[k][m][r] = N[r];
      mt.D1[k][m][r] = dN[r] * h;
    }
  }
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  int nact = n1[0] * n1[1] * n1[2];
  if (tid == 0) {
    mt.nact = nact;
    mt.rational = c_ip.mweights != nullptr;
  }
  for (int idx = tid; idx < nact * D; idx += nthr) {
    int ra = idx / D, a = idx % D;
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    int64_t cp = 0;
    for (int k = D - 1; k >= 0; --k) {
      int s = mspan[c_ip.soff[k] + e[k]];
      cp = cp * c_ip.mn[k] + (s - c_ip.pm[k] + r[k]);
    }
    mt.P[idx] = ctrl[cp * D + a];
    if (a == 0) mt.Wt[ra] = c_ip.mweights ? c_ip.mweights[cp] : 1.0;
  }
}

// NURBS (NEXT N4): W = Σ_r w_r N_r and ∂_β W at sample node m (B-spline: 1, 0)
template <int D>
__device__ void macro_W(const InterpConst &c_ip, const MacroTile<D> &mt, int m, double &W, double dW[D]) {
  W = 1.0;
  for (int be = 0; be < D; ++be) dW[be] = 0.0;
  if (!mt.rational) return;
  const int mm[3] = {m % c_ip.mv[0], (m / c_ip.mv[0]) % c_ip.mv[1], m / (c_ip.mv[0] * c_ip.mv[1])};
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  W = 0.0;
  for (int ra = 0; ra < mt.nact; ++ra) {
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    double N = 1.0;
    for (int k = 0; k < D; ++k) N *= mt.B1[k][mm[k]][r[k]];
    W += mt.Wt[ra] * N;
    for (int be = 0; be < D; ++be) {
      double v = 1.0;
      for (int k = 0; k < D; ++k) v *= (k == be) ? mt.D1[k][mm[k]][r[k]] : mt.B1[k][mm[k]][r[k]];
      dW[be] += mt.Wt[ra] * v;
    }
  }
}

// ∂R_r/∂ξ_β at sample node m (rational: w_r (∂_β N_r W - N_r ∂_β W) / W²)
template <int D>
__device__ __forceinline__ void basis_grad(const InterpConst &c_ip, const MacroTile<D> &mt, int m, int ra, double W,
                                           const double *dW, double g[D]) {
  const int mm[3] = {m % c_ip.mv[0], (m / c_ip.mv[0]) % c_ip.mv[1], m / (c_ip.mv[0] * c_ip.mv[1])};
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
  double N = 1.0;
  for (int k = 0; k < D; ++k) N *= mt.B1[k][mm[k]][r[k]];
  for (int be = 0; be < D; ++be) {
    double v = 1.0;
    for (int k = 0; k < D; ++k) v *= (k == be) ? mt.D1[k][mm[k]][r[k]] : mt.B1[k][mm[k]][r[k]];
    g[be] = mt.rational ? mt.Wt[ra] * (v * W - N * dW[be]) / (W * W) : v;
  }
}

// J[a][β] = ∂F_a/∂ξ_β at tensor sample node m (m^d nodes, direction-0 fastest)
template <int D>
__device__ void macro_J(const InterpConst &c_ip, const MacroTile<D> &mt, int m, double J[D][D]) {
  const int mm[3] = {m % c_ip.mv[0], (m / c_ip.mv[0]) % c_ip.mv[1], m / (c_ip.mv[0] * c_ip.mv[1])};
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  for (int a = 0; a < D; ++a)
    for (int b = 0; b < D; ++b) J[a][b] = 0.0;
  double W = 1.0, dW[D];
  if (mt.rational) macro_W<D>(c_ip, mt, m, W, dW);
  for (int ra = 0; ra < mt.nact; ++ra) {
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    double g[D];
    if (mt.rational) {
      basis_grad<D>(c_ip, mt, m, ra, W, dW, g);
    } else {
      for (int be = 0; be < D; ++be) {
        double v = 1.0;
        for (int k = 0; k < D; ++k) v *= (k == be) ? mt.D1[k][mm[k]][r[k]] : mt.B1[k][mm[k]][r[k]];
        g[be] = v;
      }
    }
    for (int a = 0; a < D; ++a) {
      double x = mt.P[ra * D + a];
      for (int be = 0; be < D; ++be) J[a][be] += x * g[be];
    }
  }
}

// column β of J at sample node m for a B-spline macro tile: col[a] = Σ_r P_r[a] ∂_β N_r
template <int D>
__device__ __forceinline__ void macro_Jcol_bspline(const InterpConst &c_ip, const MacroTile<D> &mt, int m, int be,
                                                   double col[D]) {
  const int mm[3] = {m % c_ip.mv[0], (m / c_ip.mv[0]) % c_ip.mv[1], m / (c_ip.mv[0] * c_ip.mv[1])};
  const int n0 = c_ip.pm[0] + 1, n1 = c_ip.pm[1] + 1, n2 = D == 3 ? c_ip.pm[2] + 1 : 1;
  const double *F0 = be == 0 ? mt.D1[0][mm[0]] : mt.B1[0][mm[0]];
  const double *F1 = be == 1 ? mt.D1[1][mm[1]] : mt.B1[1][mm[1]];
  const double *F2 = be == D - 1 && D == 3 ? mt.D1[D - 1][mm[D - 1]] : mt.B1[D - 1][mm[D - 1]];
#pragma unroll
  for (int a = 0; a < D; ++a) col[a] = 0.0;
  const double *P = mt.P;
  for (int r2 = 0; r2 < n2; ++r2) {
    const double f2 = D == 3 ? F2[r2] : 1.0;
    for (int r1 = 0; r1 < n1; ++r1) {
      const double f12 = F1[r1] * f2;
      for (int r0 = 0; r0 < n0; ++r0, P += D) {
        const double g = F0[r0] * f12;
#pragma unroll
        for (int a = 0; a < D; ++a) col[a] = fma(P[a], g, col[a]);
      }
    }
  }
}

__device__ __forceinline__ void lame(double E, double nu, double &lam, double &mu) {
  lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  mu = E / (2.0 * (1.0 + nu));
}

// one 1D pass of the projection along direction `dir` of an n[0]×n[1]×n[2] array of
// NCOMP-vectors in shared memory: forward (samples -> coefficients) out[..c..] =
// Σ_i Π1[dir][c][i] in[..i..] (n[dir]: m_dir -> q_dir+1); transposed out[..i..] =
// Σ_c Π1[dir][c][i] in[..c..] (n[dir]: q_dir+1 -> m_dir).  Updates n[] to the output shape.
template <int NCOMP>
__device__ void proj_pass(const InterpConst &c_ip, const double *in, double *out, int n[3], int dir, bool transpose) {
  const int q1 = c_ip.qv[dir] + 1, m1 = c_ip.mv[dir];
  const double *Pi1 = c_ip.Pi1[dir];
  const int nin = n[dir], nout = transpose ? m1 : q1;
  int o[3] = {n[0], n[1], n[2]};
  o[dir] = nout;
  const int stride_in = dir == 0 ? 1 : (dir == 1 ? n[0] : n[0] * n[1]);
  const int stride_out = dir == 0 ? 1 : (dir == 1 ? o[0] : o[0] * o[1]);
  const int total = o[0] * o[1] * o[2];
  for (int idx = threadIdx.x; idx < total * NCOMP; idx += blockDim.x) {
    const int C = idx / NCOMP, comp = idx - C * NCOMP;
    const int c = (C / stride_out) % nout;
    const int rest = C - c * stride_out;                         // other indices, output strides
    const int hi = rest / (stride_out * nout), lo = rest % stride_out;
    const double *src = in + ((hi * nin) * stride_in + lo) * NCOMP + comp;
    double acc = 0.0;
    for (int k = 0; k < nin; ++k)
      acc = fma(transpose ? Pi1[k * m1 + c] : Pi1[c * m1 + k], src[k * stride_in * NCOMP], acc);
    out[idx] = acc;
  }
  n[dir] = nout;
}

// the isotropic m = q+1 case with every index a compile-time constant
template <int D, int Q, int DIR, bool TRANSPOSE, int NCOMP>
__device__ __forceinline__ void tensor_pass(const InterpConst &c_ip, const double *in, double *out) {
  constexpr int Q1 = Q + 1, NPI = D == 2 ? Q1 * Q1 : Q1 * Q1 * Q1;
  constexpr int STRIDE = DIR == 0 ? 1 : (DIR == 1 ? Q1 : Q1 * Q1);
  const double *Pi1 = c_ip.Pi1[DIR];
  for (int idx = threadIdx.x; idx < NPI * NCOMP; idx += blockDim.x) {
    const int C = idx / NCOMP, comp = idx - C * NCOMP;
    const int c = (C / STRIDE) % Q1;
    const double *src = in + (C - c * STRIDE) * NCOMP + comp;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < Q1; ++k)
      acc = fma(TRANSPOSE ? Pi1[k * Q1 + c] : Pi1[c * Q1 + k], src[k * STRIDE * NCOMP], acc);
    out[idx] = acc;
  }
}

template <int D, int Q, bool TRANSPOSE, int NCOMP>
__device__ const double *tensor_apply(const InterpConst &c_ip, double *a, double *b) {
  tensor_pass<D, Q, 0, TRANSPOSE, NCOMP>(c_ip, a, b);
  __syncthreads();
  tensor_pass<D, Q, 1, TRANSPOSE, NCOMP>(c_ip, b, a);
  __syncthreads();
  if (D == 2) return a;
  tensor_pass<D, Q, 2, TRANSPOSE, NCOMP>(c_ip, a, b);
  __syncthreads();
  return b;
}

// all d passes; a, b: the two buffers; returns the one holding the result
template <int D, int NCOMP>
__device__ const double *proj_apply(const InterpConst &c_ip, double *a, double *b, bool transpose) {
  int n[3] = {1, 1, 1};
  for (int k = 0; k < D; ++k) n[k] = transpose ? c_ip.qv[k] + 1 : c_ip.mv[k];
  double *in = a, *out = b;
  for (int dir = 0; dir < D; ++dir) {
    proj_pass<NCOMP>(c_ip, in, out, n, dir, transpose);
    __syncthreads();
    double *t = in; in = out; out = t;
  }
  return in;
}

// per-node geometry: G = J⁻¹ (rows ǧ_i), det J, gg = G Gᵀ
template <int D>
struct NodeGeo {
  double G[D][D], gg[D][D], det;
  double W, dW[D];   // NURBS denominator and its gradient at the node (B-spline: 1, 0)
};

template <int D>
__device__ __forceinline__ void node_geometry(const InterpConst &c_ip, const MacroTile<D> &mt, NodeGeo<D> *geo,
                                              int64_t t, int *flag) {
  const int ns = c_ip.ns;
  for (int m = threadIdx.x; m < ns; m += blockDim.x) {
    double J[D][D], G[D][D];
    macro_J<D>(c_ip, mt, m, J);
    const double det = det_inv<D>(J, G);
    if (!(det > 0.0)) raise_flag(flag, 2, (int)t, m);
    NodeGeo<D> &o = geo[m];
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        o.G[i][j] = G[i][j];
        double v = 0.0;
        for (int c = 0; c < D; ++c) v += G[i][c] * G[j][c];
        o.gg[i][j] = v;
      }
    o.det = det;
    macro_W<D>(c_ip, mt, m, o.W, o.dW);
  }
}

// K2: thread = (tile, component) — a distinct symmetric / antisymmetric half (SYM, the K3
// operand) or an Ā component (i,j,a,b) (iga_interpolate); TPB tiles per CTA.  Phases: macro
// data per tile -> ∇F columns (one thread per node and direction) -> det / J⁻¹ per node ->
// each thread evaluates its component (Eq. 37, closed form) at the (q+1)^d nodes into
// registers, applies (V1⁻¹)^{⊗d} by D in-place 1D passes (all indices compile-time) and
// writes its (q+1)^d interpolation coefficients.
template <int D, int Q, bool SYM = false>
struct K2Shape {
  static constexpr int Q1 = Q + 1, NPI = D == 2 ? Q1 * Q1 : Q1 * Q1 * Q1, DD = D * D, NC = DD * DD;
  // SYM (the K3 operand of the Eq. 38-reduced contraction): one thread per distinct
  // component, n_p1² symmetric + n_p2² antisymmetric (45 in 3D, 10 in 2D); else all d⁴
  static constexpr int NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2, NS = NP1 * NP1 + NP2 * NP2;
  static constexpr int NT = SYM ? NS : NC;
  static constexpr int TPB = D == 2 ? (Q <= 2 ? 16 : 8) : 4;   // tiles per CTA (static shared memory < 48 KB)
  static constexpr int THREADS = TPB * NT;
  static constexpr bool REG = NPI <= 27;        // register path; larger q: shared-memory passes
};

// Ā_ij[a,b] at a node (Eq. 37, closed form)
template <int D>
__device__ __forceinline__ double abar(const NodeGeo<D> &g, double lam, double mu, int i, int j, int a, int b) {
  return g.det * (lam * g.G[i][a] * g.G[j][b] + mu * g.G[j][a] * g.G[i][b] + (a == b ? mu * g.gg[i][j] : 0.0));
}

// the K3 B operand of the Eq. 38-reduced contraction: symmetric part
// ½(⟨Ā_ij[a,b]⟩ + ⟨Ā_ij[b,a]⟩) of P1 pair p = (i,j) at output o = (a,b), a <= b (column
// p·n_π + C, block row o·tpc + tl), antisymmetric part ½(⟨Ā_ij[a,b]⟩ − ⟨Ā_ij[b,a]⟩) of P2 pair
// (column k1 + p'·n_π + C, block row (n_p1 + o')·tpc + tl).  comp < n_p1²: (p, o); else (p', o').
template <int D>
__device__ __forceinline__ void sym_component(int comp, bool &part2, int &i, int &j, int &a, int &b, int &p, int &o) {
  constexpr int NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2;
  part2 = comp >= NP1 * NP1;
  if (!part2) {
    p = comp / NP1;
    o = comp % NP1;
    sym_pair(D, p, i, j);
    sym_pair(D, o, a, b);
  } else {
    const int c2 = comp - NP1 * NP1;
    p = c2 / NP2;
    o = c2 % NP2;
    anti_pair(D, p, i, j);
    anti_pair(D, o, a, b);
  }
}

// FM offset of the sym-layout K3 B operand entry (tile t, block row o_col, column k)
__device__ __forceinline__ int64_t sym_b_index(int64_t t, int o_col, int k, int tpc, int ks3) {
  const int64_t nb = t / tpc;
  const int rr = o_col * tpc + (int)(t - nb * tpc);
  return (nb * (ks3 / 16) + (k >> 4)) * (int64_t)(IGA_GEMM_BN * 16) + (rr & ~7) * 16 + ((k >> 2) & 3) * 32 +
         ((rr & 7) << 2) + (k & 3);
}

template <int D, int Q, bool SYM>
__global__ void __launch_bounds__(K2Shape<D, Q, SYM>::THREADS)
k2_interpolate(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
               const int *__restrict__ mspan, const double *__restrict__ young, int ypt,
               double nu, double *__restrict__ coef, int kstride, int k1, int tpc, int64_t n_tiles, int *flag) {
  using S = K2Shape<D, Q, SYM>;
  static_assert(S::REG, "register path only for (q+1)^d <= 27");
  constexpr int Q1 = S::Q1, NPI = S::NPI, DD = S::DD, NT = S::NT, TPB = S::TPB;
  __shared__ MacroTile<D> mt[TPB];
  __shared__ NodeGeo<D> geo[TPB][NPI];
  // tile fastest: the TPB threads of one component write its coefficients of TPB neighbouring
  // tiles, which the fragment-major layout puts 32 B apart (one 128-B line per component and C
  // in 3D) — 4× fewer L2 write requests than one component per lane
  const int tl = threadIdx.x % TPB, comp = threadIdx.x / TPB;
  const int64_t t = (int64_t)blockIdx.x * TPB + tl;
  const bool live = t < n_tiles;
  const int64_t tg = t + c_ip.t_base;   // global tile id (macro element, E, error report)
  if (live) load_macro_tile<D>(c_ip, mt[tl], tg, ctrl, mknots, mspan, comp, NT);
  __syncthreads();
  // ∇F at the nodes: B-spline maps one column J[:, β] per thread (NPI·D threads of the
  // tile, staged in the node's G slot), then det / J⁻¹ per node; NURBS maps the whole
  // quotient-rule J per node
  if (live && !mt[tl].rational)
    for (int w = comp; w < NPI * D; w += NT) {
      const int m = w / D, be = w % D;
      double col[D];
      macro_Jcol_bspline<D>(c_ip, mt[tl], m, be, col);
#pragma unroll
      for (int a = 0; a < D; ++a) geo[tl][m].G[a][be] = col[a];
    }
  __syncthreads();
  if (live)
    for (int m = comp; m < NPI; m += NT) {
      double J[D][D], G[D][D];
      if (mt[tl].rational) macro_J<D>(c_ip, mt[tl], m, J);
      else
        for (int a = 0; a < D; ++a)
          for (int be = 0; be < D; ++be) J[a][be] = geo[tl][m].G[a][be];
      const double det = det_inv<D>(J, G);
      if (!(det > 0.0)) raise_flag(flag, 2, (int)tg, m);
      NodeGeo<D> &o = geo[tl][m];
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
          o.G[i][j] = G[i][j];
          double v = 0.0;
          for (int c = 0; c < D; ++c) v += G[i][c] * G[j][c];
          o.gg[i][j] = v;
        }
      o.det = det;
    }
  __syncthreads();
  if (!live) return;
  double lam, mu;
  lame(young[ypt ? tg : 0], nu, lam, mu);
  double x[NPI];
  int i, j, a, b, ij = 0, ab = 0, p = 0, o = 0;
  bool part2 = false;
  if (SYM) {
    sym_component<D>(comp, part2, i, j, a, b, p, o);
#pragma unroll
    for (int m = 0; m < NPI; ++m) {
      const double xab = abar<D>(geo[tl][m], lam, mu, i, j, a, b);
      const double xba = a == b ? xab : abar<D>(geo[tl][m], lam, mu, i, j, b, a);
      x[m] = 0.5 * (part2 ? xab - xba : xab + xba);
    }
  } else {
    ij = comp / DD;
    ab = comp % DD;
    i = ij / D;
    j = ij % D;
    a = ab / D;
    b = ab % D;
#pragma unroll
    for (int m = 0; m < NPI; ++m) x[m] = abar<D>(geo[tl][m], lam, mu, i, j, a, b);
  }
  // direction 0, 1 (, 2), in place one line of Q1 values at a time (few live registers):
  // out[c] = Σ_m Π1[dir][c][m] in[m] along the direction
#pragma unroll
  for (int dir = 0; dir < D; ++dir) {
    constexpr int L = NPI / Q1;
    const int stride = dir == 0 ? 1 : (dir == 1 ? Q1 : Q1 * Q1);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int base = dir == 0 ? l * Q1 : (dir == 1 ? (l % Q1) + (l / Q1) * Q1 * Q1 : l);
      double v[Q1];
#pragma unroll
      for (int m = 0; m < Q1; ++m) v[m] = x[base + m * stride];
#pragma unroll
      for (int c = 0; c < Q1; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < Q1; ++m) acc = fma(c_ip.Pi1[dir][c * Q1 + m], v[m], acc);
        x[base + c * stride] = acc;
      }
    }
  }
  if (SYM) {
    // the sym-layout K3 B operand (row part hoisted, 32-bit column offsets)
    const int o_col = part2 ? D * (D + 1) / 2 + o : o;
    const int kb = part2 ? k1 + p * NPI : p * NPI;
    double *base = coef + sym_b_index(t, o_col, 0, tpc, kstride);
#pragma unroll
    for (int C = 0; C < NPI; ++C) {
      const int k = kb + C;
      base[(k >> 4) * (IGA_GEMM_BN * 16) + ((k >> 2) & 3) * 32 + (k & 3)] = x[C];
    }
  } else {   // full coefficients, row-major coef[(t*DD + ab)*kstride + ij*npi + C] (iga_interpolate)
    const int64_t n = t * DD + ab;
#pragma unroll
    for (int C = 0; C < NPI; ++C) coef[n * kstride + ij * NPI + C] = x[C];
  }
}

// shared memory of the one-CTA-per-tile K2 projection path: two ns×d⁴ buffers and the ns
// node geometries, ns = Π m_k
size_t macro_smem_bytes(int d, int ns_) {
  const size_t ns = (size_t)ns_, nc = (size_t)d * d * d * d;
  const size_t geo = d == 2 ? sizeof(NodeGeo<2>) : sizeof(NodeGeo<3>);
  return sizeof(double) * 2 * ns * nc + ns * geo;
}

// K5b: each of its two buffers holds ns×d⁴ doubles (W', Ŵ) or the tile's staged Y
__host__ __device__ inline size_t k5b_buf_doubles(int d, int ns, int k5s, int k5kap) {
  const size_t nc = (size_t)d * d * d * d, np1 = d * (d + 1) / 2, np2 = d * (d - 1) / 2;
  const size_t ny = np1 * k5s + np2 * (size_t)(k5kap - k5s), nw = (size_t)ns * nc;
  return ny > nw ? ny : nw;
}

// K5b dynamic shared memory: two buffers, ∂S/∂J (ns×d²), the node geometries, the gphys groups
size_t k5b_smem_bytes(const Handle &h, int ns) {
  const size_t geo = h.d == 2 ? sizeof(NodeGeo<2>) : sizeof(NodeGeo<3>);
  return sizeof(double) * (2 * k5b_buf_doubles(h.d, ns, h.k5_split, h.k5_kap) + (size_t)ns * h.d * h.d) + ns * geo +
         sizeof(int) * (size_t)(h.k5_kap / 8);
}

// compile-time n_π for an isotropic degree Q; Q = -1: anisotropic (runtime c_ip.npi)
template <int D, int Q>
__device__ __forceinline__ int npi_of(const InterpConst &c_ip) {
  if constexpr (Q >= 0) return D == 2 ? (Q + 1) * (Q + 1) : (Q + 1) * (Q + 1) * (Q + 1);
  else return c_ip.npi;
}

// Ŵ = Πᵀ W or coef = Π samples: compile-time passes when isotropic with m = q+1
template <int D, int Q, bool TRANSPOSE, int NCOMP>
__device__ const double *apply_projection(const InterpConst &c_ip, double *a, double *b) {
  if constexpr (Q >= 0) {
    if (c_ip.iso && c_ip.m == Q + 1) return tensor_apply<D, Q, TRANSPOSE, NCOMP>(c_ip, a, b);
  }
  return proj_apply<D, NCOMP>(c_ip, a, b, TRANSPOSE);
}

// K2 for (q+1)^d > 27, an L2 projection with m > q+1 points or anisotropic degrees (NEXT
// N2): one CTA per tile, Ā sampled at the Π m_k Gauss nodes into shared memory, d passes.
template <int D, int Q>
__global__ void __launch_bounds__(256)
k2_interpolate_smem(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl,
                    const double *__restrict__ mknots, const int *__restrict__ mspan, const double *__restrict__ young,
                    int ypt, double nu, double *__restrict__ coef, int kstride, int fm, int k1, int tpc,
                    int64_t n_tiles, int *flag) {
  constexpr int DD = D * D, NC = DD * DD;
  const int NPI = npi_of<D, Q>(c_ip), NK = DD * NPI;
  const int ns = c_ip.ns;
  extern __shared__ double dyn[];
  double *S0 = dyn, *S1 = dyn + (size_t)ns * NC;
  NodeGeo<D> *geo = reinterpret_cast<NodeGeo<D> *>(dyn + 2 * (size_t)ns * NC);
  __shared__ MacroTile<D> mt;
  const int64_t t = blockIdx.x, tg = t + c_ip.t_base;
  load_macro_tile<D>(c_ip, mt, tg, ctrl, mknots, mspan);
  __syncthreads();
  node_geometry<D>(c_ip, mt, geo, tg, flag);
  double lam, mu;
  lame(young[ypt ? tg : 0], nu, lam, mu);
  __syncthreads();
  for (int it = threadIdx.x; it < ns * DD; it += blockDim.x) {   // Ā (Eq. 37, closed form)
    const int m = it / DD, ij = it % DD, i = ij / D, j = ij % D;
    const NodeGeo<D> &g = geo[m];
    double *o = S0 + m * NC + ij * DD;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        o[a * D + b] = g.det * (lam * g.G[i][a] * g.G[j][b] + mu * g.G[j][a] * g.G[i][b] + (a == b ? mu * g.gg[i][j] : 0.0));
  }
  __syncthreads();
  const double *res = apply_projection<D, Q, false, NC>(c_ip, S0, S1);
  for (int idx = fm ? DD * NK : threadIdx.x; idx < DD * NK; idx += blockDim.x) {   // full (iga_interpolate)
    const int ab = idx / NK, kap = idx % NK, ij = kap / NPI, C = kap % NPI;
    const int64_t n = t * DD + ab;
    if (!fm) coef[n * kstride + kap] = res[C * NC + ij * DD + ab];
  }
  if (!fm) return;
  // the sym-layout K3 B operand (Eq. 38-reduced contraction)
  constexpr int NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2, NS = NP1 * NP1 + NP2 * NP2;
  for (int idx = threadIdx.x; idx < NS * NPI; idx += blockDim.x) {
    const int comp = idx / NPI, C = idx % NPI;
    bool part2;
    int i, j, a, b, p, o;
    sym_component<D>(comp, part2, i, j, a, b, p, o);
    const double *r = res + C * NC + (i * D + j) * DD;
    const double v = 0.5 * (part2 ? r[a * D + b] - r[b * D + a] : r[a * D + b] + r[b * D + a]);
    const int o_col = part2 ? NP1 + o : o, k = part2 ? k1 + p * NPI + C : p * NPI + C;
    coef[sym_b_index(t, o_col, k, tpc, kstride)] = a == b && !part2 ? r[a * D + a] : v;
  }
}

// K5b tail (both variants): the reverse mode of S = ⟨Ŵ, Ā(J)⟩ at the ns nodes from Ŵ
// (Wh_all[m·d⁴ + ij·d² + ab]) and the node geometries, ∂S/∂J, the chain to the active
// control points.  Sp, Qm: ns·d² doubles of scratch each.
template <int D>
__device__ void k5b_tail(const InterpConst &c_ip, const MacroTile<D> &mt, const NodeGeo<D> *geo, const double *Wh_all,
                         double *Sp, double *Qm, double *dSdJ, double lam, double mu, int64_t t,
                         double *__restrict__ gpart) {
  constexpr int DD = D * D, NC = DD * DD;
  const int ns = c_ip.ns;
  // reverse mode of S = ⟨Ŵ, Ā(J)⟩ per node, one thread per (node m, i, n):
  // Sp = the (i, n) part of S / det, Q[i][n] = det (λ d1 + μ d2 + μ d3)
  for (int it = threadIdx.x; it < ns * DD; it += blockDim.x) {
    const int m = it / DD, mi = (it % DD) / D, n = it % D;
    const double *Wh = Wh_all + m * NC;   // Ŵ[ij*DD + ab]
    const NodeGeo<D> &g = geo[m];
    double sp = 0.0, d1 = 0, d2 = 0, d3 = 0, sd = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      sd += Wh[(mi * D + n) * DD + a * D + a];
#pragma unroll
      for (int b = 0; b < D; ++b) {
        const double x = Wh[(mi * D + n) * DD + a * D + b];
        sp = fma(x, lam * g.G[mi][a] * g.G[n][b] + mu * g.G[n][a] * g.G[mi][b], sp);
      }
    }
    sp = fma(mu * sd, g.gg[mi][n], sp);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double wmj = 0.0, wjm = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) {
        const double Gjb = g.G[j][b];
        d1 = fma(Wh[(mi * D + j) * DD + n * D + b] + Wh[(j * D + mi) * DD + b * D + n], Gjb, d1);
        d2 = fma(Wh[(j * D + mi) * DD + n * D + b] + Wh[(mi * D + j) * DD + b * D + n], Gjb, d2);
        wmj += Wh[(mi * D + j) * DD + b * D + b];
        wjm += Wh[(j * D + mi) * DD + b * D + b];
      }
      d3 = fma(wmj + wjm, g.G[j][n], d3);
    }
    Sp[it] = sp;
    Qm[it] = g.det * (lam * d1 + mu * d2 + mu * d3);
  }
  __syncthreads();
  // ∂S/∂J[a][β] = S G[β][a] - Σ_{i,n} G[i][a] Q[i][n] G[β][n], one thread per (m, a, β)
  for (int it = threadIdx.x; it < ns * DD; it += blockDim.x) {
    const int m = it / DD, a = (it % DD) / D, be = it % D;
    const NodeGeo<D> &g = geo[m];
    double S = 0.0;
#pragma unroll
    for (int x = 0; x < DD; ++x) S += Sp[m * DD + x];
    double v = g.det * S * g.G[be][a];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int n = 0; n < D; ++n) v -= g.G[i][a] * Qm[m * DD + i * D + n] * g.G[be][n];
    dSdJ[it] = v;
  }
  __syncthreads();
  // chain to the active control points: g[r][a] = Σ_m Σ_β ∂S/∂J[a][β] ∂_β R_r(ξ_m)
  // (node indices (m0, m1, m2) stepped, no divisions in the node loop)
  for (int idx = threadIdx.x; idx < mt.nact * D; idx += blockDim.x) {
    const int ra = idx / D, a = idx % D;
    const int n0 = c_ip.pm[0] + 1, n1 = D > 1 ? c_ip.pm[1] + 1 : 1;
    const int r[3] = {ra % n0, (ra / n0) % n1, ra / (n0 * n1)};
    double acc = 0.0;
    int mm[3] = {0, 0, 0};
    for (int m = 0; m < ns; ++m) {
      double g[D];
      if (mt.rational) {
        basis_grad<D>(c_ip, mt, m, ra, geo[m].W, geo[m].dW, g);
      } else {
        double bv[D], dv[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          bv[k] = mt.B1[k][mm[k]][r[k]];
          dv[k] = mt.D1[k][mm[k]][r[k]];
        }
        g[0] = D == 2 ? dv[0] * bv[1] : dv[0] * bv[1] * bv[D - 1];
        g[1] = D == 2 ? bv[0] * dv[1] : bv[0] * dv[1] * bv[D - 1];
        if (D == 3) g[D - 1] = bv[0] * bv[1] * dv[D - 1];
      }
#pragma unroll
      for (int be = 0; be < D; ++be) acc = fma(dSdJ[m * DD + a * D + be], g[be], acc);
      if (++mm[0] == c_ip.mv[0]) {
        mm[0] = 0;
        if (++mm[1] == c_ip.mv[1]) { mm[1] = 0; ++mm[2]; }
      }
    }
    gpart[((size_t)t * mt.nact + ra) * D + a] = acc;
  }
}

// K5b: one CTA per tile: Ŵ = Πᵀ W at the m^d sample nodes, reverse mode of
// S = ⟨Ŵ, Ā(J)⟩ per node, chain to the active macro control points.
#ifndef IGA_K5B_THREADS
#define IGA_K5B_THREADS 128   // per tile; several tiles' CTAs per SM overlap the per-node phase
#endif
template <int D, int Q>
__global__ void __launch_bounds__(IGA_K5B_THREADS)
k5b_reverse(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
            const int *__restrict__ mspan, const double *__restrict__ young, int ypt, double nu,
            const double *__restrict__ W, int ldw, int tpc, int k5s, int k5kap, const int32_t *__restrict__ gphys,
            double *__restrict__ gpart, int *flag) {
  constexpr int DD = D * D, NC = DD * DD, NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2;
  const int NPI = npi_of<D, Q>(c_ip);
  const int ns = c_ip.ns, k2n = k5kap - k5s;
  const size_t nbuf = k5b_buf_doubles(D, ns, k5s, k5kap);
  extern __shared__ double dyn[];
  double *S0 = dyn, *S1 = dyn + nbuf, *dSdJ = dyn + 2 * nbuf;
  NodeGeo<D> *geo = reinterpret_cast<NodeGeo<D> *>(dSdJ + (size_t)ns * DD);
  int *sgp = reinterpret_cast<int *>(geo + ns);   // gphys of the k5kap/8 logical groups
  __shared__ MacroTile<D> mt;
  const int64_t t = blockIdx.x, tg = t + c_ip.t_base;
  load_macro_tile<D>(c_ip, mt, tg, ctrl, mknots, mspan);
  for (int g = threadIdx.x; g < k5kap / 8; g += blockDim.x) sgp[g] = gphys[g];
  __syncthreads();
  // stage this tile's Y (K5g/K5a output) compactly, coalesced: Y⁺[o][κ] (o < NP1, κ < k5s),
  // then Y⁻[o][κ - k5s]; 8 consecutive threads read one 64-byte physical row group
  const int64_t nbk = t / tpc;
  const int tl = (int)(t - nbk * tpc);
  const double *Wt = W + (size_t)(nbk * IGA_GEMM_BN + tl) * ldw;
  const int n1 = NP1 * k5s;
#pragma unroll
  for (int o = 0; o < NP1 + NP2; ++o) {
    const bool p2 = o >= NP1;
    const int len = p2 ? k2n : k5s, k0 = p2 ? k5s : 0;
    double *dst = S1 + (p2 ? n1 + (o - NP1) * k2n : o * k5s);
    const double *src = Wt + (size_t)(o * tpc) * ldw;
    for (int r = threadIdx.x; r < len; r += blockDim.x) {
      const int kap = k0 + r;
      dst[r] = src[sgp[kap >> 3] * 8 + (kap & 7)];
    }
  }
  __syncthreads();
  // W' from Y (Eq. 38-reduced contraction): ⟨W', Ā⟩ = Σ Y⁺ Ā⁺' + Σ Y⁻ Ā⁻'
  // with Ā^±'_ij[a,b] = ½(Ā_ij[a,b] ± Ā_ij[b,a]) for i <= j, so W'_ij[a,b] = ½Y⁺_ij[ab]
  // (Y⁺_ij[aa] on the diagonal) ± ½Y⁻_ij[ab] (i < j, + for a < b), W'_ij = 0 for i > j
  for (int idx = threadIdx.x; idx < NC * NPI; idx += blockDim.x) {
    const int C = idx / NC, comp = idx % NC, ij = comp / DD, ab = comp % DD;
    const int i = ij / D, j = ij % D, a = ab / D, b = ab % D;
    double w = 0.0;
    if (i <= j) {
      const int lo = min(a, b), hi = max(a, b);
      const double y1 = S1[sym_index(D, lo, hi) * k5s + sym_index(D, i, j) * NPI + C];
      w = a == b ? y1 : 0.5 * y1;
      if (i < j && a != b) {
        const double y2 = S1[n1 + anti_index(D, lo, hi) * k2n + anti_index(D, i, j) * NPI + C];
        w = fma(a < b ? 0.5 : -0.5, y2, w);
      }
    }
    S0[C * NC + comp] = w;
  }
  __syncthreads();
  node_geometry<D>(c_ip, mt, geo, tg, flag);
  // Ŵ = Πᵀ W (also syncs geo)
  const double *Wh_all = apply_projection<D, Q, true, NC>(c_ip, S0, S1);
  double *Sp = Wh_all == S0 ? S1 : S0, *Qm = Sp + (size_t)ns * DD;   // the free buffer
  double lam, mu;
  lame(young[ypt ? tg : 0], nu, lam, mu);
  k5b_tail<D>(c_ip, mt, geo, Wh_all, Sp, Qm, dSdJ, lam, mu, t, gpart);
}

// K5b register path (isotropic q, m = q+1, (q+1)^d <= 27; the bench shapes): one CTA per
// tile in two roles.  Y role (warps 0-1): thread = one of the 45 (3D) / 10 (2D) distinct
// components of Y, its n_π values loaded straight into registers (all loads in flight at
// once), Ŷ = Πᵀ Y by d in-place register passes (Πᵀ is linear per component, so it
// commutes with the W' expansion below), Ŷ to shared memory.  Geometry role (warps 2-3):
// macro data, ∇F columns, det / J⁻¹ per node, overlapping the Y loads.  Then Ŵ' per node
// from Ŷ and the common tail.
#define IGA_K5B_YT 64   // threads of the Y role (>= 45)
__device__ __forceinline__ void macro_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

template <int D, int Q>
__global__ void __launch_bounds__(IGA_K5B_THREADS)
k5b_reverse_reg(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
                const int *__restrict__ mspan, const double *__restrict__ young, int ypt, double nu,
                const double *__restrict__ W, int ldw, int tpc, int k5s, const int32_t *__restrict__ gphys,
                double *__restrict__ gpart, int *flag) {
  constexpr int Q1 = Q + 1, NPI = D == 2 ? Q1 * Q1 : Q1 * Q1 * Q1, DD = D * D, NC = DD * DD;
  constexpr int NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2, NS = NP1 * NP1 + NP2 * NP2;
  constexpr int GT = IGA_K5B_THREADS - IGA_K5B_YT;   // geometry-role threads
  static_assert(NS <= IGA_K5B_YT && GT >= 32, "K5b role split");
  __shared__ MacroTile<D> mt;
  __shared__ NodeGeo<D> geo[NPI];
  __shared__ double Yh[NPI][NS + 1];   // Ŷ[node][component]
  __shared__ double Wh[NPI * NC];      // Ŵ'[node][ij·d² + ab]
  __shared__ double SQ[2 * NPI * DD];  // Sp, Qm of the tail
  __shared__ double dSdJ[NPI * DD];
  const int tid = threadIdx.x;
  const int64_t t = blockIdx.x, tg = t + c_ip.t_base;
  if (tid < IGA_K5B_YT) {
    if (tid < NS) {
      bool part2;
      int i, j, a, b, p, o;
      sym_component<D>(tid, part2, i, j, a, b, p, o);
      const int64_t nbk = t / tpc;
      const int tl = (int)(t - nbk * tpc);
      const double *src = W + (size_t)(nbk * IGA_GEMM_BN + (part2 ? NP1 + o : o) * tpc + tl) * ldw;
      const int kb = part2 ? k5s + p * NPI : p * NPI;
      double x[NPI];
#pragma unroll
      for (int C = 0; C < NPI; ++C) {
        const int k = kb + C;
        x[C] = src[__ldg(gphys + (k >> 3)) * 8 + (k & 7)];
      }
      // Πᵀ along directions 0, 1 (, 2), in place: out[m] = Σ_c Π1[dir][c][m] in[c]
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        constexpr int L = NPI / Q1;
        const int stride = dir == 0 ? 1 : (dir == 1 ? Q1 : Q1 * Q1);
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const int base = dir == 0 ? l * Q1 : (dir == 1 ? (l % Q1) + (l / Q1) * Q1 * Q1 : l);
          double v[Q1];
#pragma unroll
          for (int c = 0; c < Q1; ++c) v[c] = x[base + c * stride];
#pragma unroll
          for (int m = 0; m < Q1; ++m) {
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < Q1; ++c) acc = fma(c_ip.Pi1[dir][c * Q1 + m], v[c], acc);
            x[base + m * stride] = acc;
          }
        }
      }
#pragma unroll
      for (int m = 0; m < NPI; ++m) Yh[m][tid] = x[m];
    }
  } else {
    const int gt = tid - IGA_K5B_YT;
    load_macro_tile<D>(c_ip, mt, tg, ctrl, mknots, mspan, gt, GT);
    macro_bar(1, GT);
    if (!mt.rational)
      for (int w = gt; w < NPI * D; w += GT) {   // ∇F column β at node m
        const int m = w / D, be = w % D;
        double col[D];
        macro_Jcol_bspline<D>(c_ip, mt, m, be, col);
#pragma unroll
        for (int a = 0; a < D; ++a) geo[m].G[a][be] = col[a];
      }
    macro_bar(1, GT);
    for (int m = gt; m < NPI; m += GT) {
      double J[D][D], G[D][D];
      if (mt.rational) macro_J<D>(c_ip, mt, m, J);
      else
        for (int a = 0; a < D; ++a)
          for (int be = 0; be < D; ++be) J[a][be] = geo[m].G[a][be];
      const double det = det_inv<D>(J, G);
      if (!(det > 0.0)) raise_flag(flag, 2, (int)tg, m);
      NodeGeo<D> &o = geo[m];
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
          o.G[i][j] = G[i][j];
          double v = 0.0;
          for (int c = 0; c < D; ++c) v += G[i][c] * G[j][c];
          o.gg[i][j] = v;
        }
      o.det = det;
      macro_W<D>(c_ip, mt, m, o.W, o.dW);
    }
  }
  __syncthreads();
  // Ŵ' from Ŷ (the W' expansion of k5b_reverse, per node): W'_ij[a,b] = ½Y⁺_ij[ab]
  // (Y⁺_ij[aa] on the diagonal) ± ½Y⁻_ij[ab] (i < j, + for a < b), 0 for i > j
  // (thread = component: its two Ŷ sources and weights once, then the n_π nodes)
  for (int comp = tid; comp < NC; comp += IGA_K5B_THREADS) {
    const int ij = comp / DD, ab = comp % DD, i = ij / D, j = ij % D, a = ab / D, b = ab % D;
    const int lo = min(a, b), hi = max(a, b);
    const int c1 = sym_index(D, i <= j ? i : 0, i <= j ? j : 0) * NP1 + sym_index(D, lo, hi);
    const double f1 = i > j ? 0.0 : (a == b ? 1.0 : 0.5);
    const bool two = i < j && a != b;
    const int c2 = two ? NP1 * NP1 + anti_index(D, i, j) * NP2 + anti_index(D, lo, hi) : c1;
    const double f2 = two ? (a < b ? 0.5 : -0.5) : 0.0;
#pragma unroll
    for (int m = 0; m < NPI; ++m) Wh[m * NC + comp] = fma(f2, Yh[m][c2], f1 * Yh[m][c1]);
  }
  __syncthreads();
  double lam, mu;
  lame(young[ypt ? tg : 0], nu, lam, mu);
  k5b_tail<D>(c_ip, mt, geo, Wh, SQ, SQ + NPI * DD, dSdJ, lam, mu, t, gpart);
}

// ---------------------------------------------------------------------------------
// Volume, volume gradient, body-force load vector (§3.1 Eqs. 14-19, Eq. 53,
// Eqs. 66-67).  Per tile: det J_ℳ at the m^d sample nodes, its
// projection coefficients d^(t) = Π·det (Eq. 15), V_t = t^h · d^(t) (Eq. 19); for the
// gradient the adjoint weights ŵ_m = (Πᵀ t^h)_m (the adjoint field of Eq. 67 at the
// samples) give ∂V_t/∂J_m = ŵ_m det J_m J_m⁻ᵀ, chained to the control points.
template <int D>
__global__ void __launch_bounds__(128)
kv_tile(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
        const int *__restrict__ mspan, const double *__restrict__ th, int npi, double *__restrict__ dcoef,
        double *__restrict__ Vt, double *__restrict__ gpart, int *flag) {
  // 3D: m <= 6 (set_projection bounds the staging of K2/K5b to m <= 5)
  constexpr int MAXNS = D == 2 ? IGA_MAXM * IGA_MAXM : 216;
  __shared__ MacroTile<D> mt;
  __shared__ double sdet[MAXNS], swh[MAXNS];
  __shared__ double sG[MAXNS][D][D];
  __shared__ double sW[MAXNS], sdW[MAXNS][D];
  __shared__ double sd[(IGA_MAXQ + 1) * (IGA_MAXQ + 1) * (IGA_MAXQ + 1)];
  const int64_t t = blockIdx.x, tg = t + c_ip.t_base;
  const int ns = c_ip.ns;
  load_macro_tile<D>(c_ip, mt, tg, ctrl, mknots, mspan);
  __syncthreads();
  for (int m = threadIdx.x; m < ns; m += blockDim.x) {
    double J[D][D], G[D][D];
    macro_J<D>(c_ip, mt, m, J);
    const double det = det_inv<D>(J, G);
    if (!(det > 0.0)) raise_flag(flag, 2, (int)tg, m);
    sdet[m] = det;
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) sG[m][i][j] = G[i][j];
    macro_W<D>(c_ip, mt, m, sW[m], sdW[m]);
  }
  __syncthreads();
  // Π[C][m] = Π_k Pi1[k][c_k][m_k]
  auto Pi = [&](int C, int m) {
    double v = 1.0;
    for (int k = 0; k < D; ++k) {
      const int q1 = c_ip.qv[k] + 1, m1 = c_ip.mv[k];
      v *= c_ip.Pi1[k][(C % q1) * m1 + m % m1];
      C /= q1;
      m /= m1;
    }
    return v;
  };
  for (int C = threadIdx.x; C < npi; C += blockDim.x) {
    double acc = 0.0;
    for (int m = 0; m < ns; ++m) acc = fma(Pi(C, m), sdet[m], acc);
    sd[C] = acc;
    dcoef[t * npi + C] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int C = 0; C < npi; ++C) v = fma(th[C], sd[C], v);
    Vt[t] = v;
  }
  if (!gpart || t >= c_ip.n_own) return;
  for (int m = threadIdx.x; m < ns; m += blockDim.x) {
    double acc = 0.0;
    for (int C = 0; C < npi; ++C) acc = fma(Pi(C, m), th[C], acc);
    swh[m] = acc * sdet[m];   // ŵ_m det_m: ∂V/∂J_m[a][β] = swh_m G_m[β][a]
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < mt.nact * D; idx += blockDim.x) {
    const int ra = idx / D, a = idx % D;
    double acc = 0.0;
    for (int m = 0; m < ns; ++m) {
      double g[D];
      basis_grad<D>(c_ip, mt, m, ra, sW[m], sdW[m], g);
      for (int be = 0; be < D; ++be) acc += swh[m] * sG[m][be][a] * g[be];
    }
    gpart[((size_t)t * mt.nact + ra) * D + a] = acc;
  }
}

// V = Σ_{owned t} V_t, fixed order (one block: strided partial sums, then a fixed tree)
__global__ void kv_sum(const double *__restrict__ Vt, int64_t n, double *__restrict__ out) {
  __shared__ double part[256];
  double acc = 0.0;
  for (int64_t t = threadIdx.x; t < n; t += 256) acc += Vt[t];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = part[0];
}

// f[i] = b Σ_{(t,A) occurrences of owned node i, fixed order} Σ_C 𝔉[A][C] d^(t)_C   (Eq. 53)
template <int D>
__global__ void __launch_bounds__(256)
kf_gather(const double *__restrict__ F, const double *__restrict__ dcoef, int npi, const int64_t *__restrict__ inv_ptr,
          const int32_t *__restrict__ inv_ent, int nl, int64_t n_nodes, double b0, double b1, double b2,
          double *__restrict__ f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  double s = 0.0;
  for (int64_t k = inv_ptr[i]; k < inv_ptr[i + 1]; ++k) {
    const int32_t e = inv_ent[k];
    const int64_t t = e / nl;
    const int A = e % nl;
    double v = 0.0;
    for (int C = 0; C < npi; ++C) v = fma(F[(size_t)A * npi + C], dcoef[t * npi + C], v);
    s += v;
  }
  const double b[3] = {b0, b1, b2};
#pragma unroll
  for (int a = 0; a < D; ++a) f[i * D + a] = b[a] * s;
}

cudaError_t launch_volume(const Handle &h, const double *ctrl, double *d_volume, double *gpart, cudaStream_t s) {
  const InterpConst ic = make_interp_const(h);
  if (h.d == 2)
    kv_tile<2><<<(unsigned)h.n_tiles, 128, 0, s>>>(ic, ctrl, h.d_mknots, h.d_mspan, h.d_th, h.npi, h.d_det, h.d_Vt,
                                                   gpart, h.d_flag);
  else
    kv_tile<3><<<(unsigned)h.n_tiles, 128, 0, s>>>(ic, ctrl, h.d_mknots, h.d_mspan, h.d_th, h.npi, h.d_det, h.d_Vt,
                                                   gpart, h.d_flag);
  cudaError_t e = cudaGetLastError();
  if (e || !d_volume) return e;
  kv_sum<<<1, 256, 0, s>>>(h.d_Vt, h.n_tiles_own, d_volume);
  return cudaGetLastError();
}

cudaError_t launch_load(const Handle &h, const double *b, double *f, cudaStream_t s) {
  const unsigned blocks = (unsigned)((h.n_nodes + 255) / 256);
  const double b2 = h.d == 3 ? b[2] : 0.0;
  if (h.d == 2)
    kf_gather<2><<<blocks, 256, 0, s>>>(h.d_F, h.d_det, h.npi, h.d_inv_ptr, h.d_inv_ent, h.n_local_ctrl, h.n_nodes,
                                        b[0], b[1], b2, f);
  else
    kf_gather<3><<<blocks, 256, 0, s>>>(h.d_F, h.d_det, h.npi, h.d_inv_ptr, h.d_inv_ent, h.n_local_ctrl, h.n_nodes,
                                        b[0], b[1], b2, f);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// A-priori projection error (Eq. 59, sampled as on P:362-364):
//   e_t = max_{ξ ∈ S} ‖Ā(ξ) − Π^H Ā(ξ)‖_F / ‖Ā(ξ)‖_F,   S = n_s^d equispaced points (R18).
// One CTA per tile.  Per component block ij (d² components a,b at a time): Ā at the
// projection nodes -> coefficients (the K2 passes) -> Π^H Ā at the samples (d evaluation
// passes with B_c^{q_k}(x_s)) -> squared differences accumulated per sample in a fixed
// order; the tile value is an exact max.  Ā ∝ E, so E = 1.
// c_ip: projection (nodes, Π1); c_sm: the same macro tile sampled at S; c_ev: evaluation
// matrices in the Pi1 slots, stored as a (n_s × (q_k+1)) "projection" (qv = n_s-1, mv = q_k+1).
template <int D>
__global__ void __launch_bounds__(256)
kp_error(const __grid_constant__ InterpConst c_ip, const __grid_constant__ InterpConst c_sm,
         const __grid_constant__ InterpConst c_ev, const double *__restrict__ ctrl, const double *__restrict__ mknots,
         const int *__restrict__ mspan, double nu, double *__restrict__ e_tile, int *flag) {
  constexpr int DD = D * D;
  const int ns = c_ip.ns, nss = c_sm.ns;
  const int nbuf = max(max(ns, c_ip.npi), nss);
  extern __shared__ double dyn[];
  double *gN = dyn;                                   // [ns][1 + DD]: det, G
  double *gS = gN + (size_t)ns * (1 + DD);            // [nss][1 + DD]
  double *S0 = gS + (size_t)nss * (1 + DD), *S1 = S0 + (size_t)nbuf * DD;
  double *num2 = S1 + (size_t)nbuf * DD, *den2 = num2 + nss;
  __shared__ MacroTile<D> mt, mts;
  __shared__ double red[256];
  const int64_t t = blockIdx.x;
  load_macro_tile<D>(c_ip, mt, t, ctrl, mknots, mspan);
  load_macro_tile<D>(c_sm, mts, t, ctrl, mknots, mspan);
  __syncthreads();
  for (int m = threadIdx.x; m < ns + nss; m += blockDim.x) {
    const bool node = m < ns;
    const int k = node ? m : m - ns;
    double J[D][D], G[D][D];
    if (node) macro_J<D>(c_ip, mt, k, J); else macro_J<D>(c_sm, mts, k, J);
    const double det = det_inv<D>(J, G);
    if (!(det > 0.0)) raise_flag(flag, 2, (int)t, k);
    double *o = (node ? gN : gS) + (size_t)k * (1 + DD);
    o[0] = det;
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) o[1 + i * D + j] = G[i][j];
    if (!node) { num2[k] = 0.0; den2[k] = 0.0; }
  }
  __syncthreads();
  double lam, mu;
  lame(1.0, nu, lam, mu);
  // Ā_ij[a,b] (Eq. 37, closed form) from (det, G)
  auto Abar = [&](const double *g, int i, int j, int a, int b) {
    const double *G = g + 1;
    double gg = 0.0;
    for (int c = 0; c < D; ++c) gg += G[i * D + c] * G[j * D + c];
    return g[0] * (lam * G[i * D + a] * G[j * D + b] + mu * G[j * D + a] * G[i * D + b] + (a == b ? mu * gg : 0.0));
  };
  for (int ij = 0; ij < DD; ++ij) {
    const int i = ij / D, j = ij % D;
    for (int it = threadIdx.x; it < ns * DD; it += blockDim.x) {
      const int m = it / DD, ab = it % DD;
      S0[it] = Abar(gN + (size_t)m * (1 + DD), i, j, ab / D, ab % D);
    }
    __syncthreads();
    double *coef = const_cast<double *>(proj_apply<D, DD>(c_ip, S0, S1, false));   // [npi][DD]
    double *other = coef == S0 ? S1 : S0;
    const double *val = proj_apply<D, DD>(c_ev, coef, other, false);                // [nss][DD]
    for (int sp = threadIdx.x; sp < nss; sp += blockDim.x) {
      const double *g = gS + (size_t)sp * (1 + DD);
      double n2 = num2[sp], d2 = den2[sp];
      for (int ab = 0; ab < DD; ++ab) {
        const double ex = Abar(g, i, j, ab / D, ab % D), df = ex - val[sp * DD + ab];
        n2 = fma(df, df, n2);
        d2 = fma(ex, ex, d2);
      }
      num2[sp] = n2;
      den2[sp] = d2;
    }
    __syncthreads();
  }
  double e = 0.0;
  for (int sp = threadIdx.x; sp < nss; sp += blockDim.x) e = fmax(e, sqrt(num2[sp]) / sqrt(den2[sp]));
  red[threadIdx.x] = e;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) e_tile[t] = red[0];
}

size_t projection_error_smem_bytes(int d, int ns, int n_s, int npi) {
  const size_t dd = (size_t)d * d, nss = d == 2 ? (size_t)n_s * n_s : (size_t)n_s * n_s * n_s;
  const size_t nbuf = std::max(std::max((size_t)ns, (size_t)npi), nss);
  return sizeof(double) * ((ns + nss) * (1 + dd) + 2 * nbuf * dd + 2 * nss);
}

cudaError_t launch_projection_error(const Handle &h, const double *ctrl, double nu, int n_s, double *e_tile,
                                    cudaStream_t s) {
  const InterpConst ic = make_interp_const(h);
  InterpConst sm = ic, ev = ic;
  int nss = 1;
  for (int k = 0; k < 3; ++k) {
    const bool act = k < h.d;
    sm.mv[k] = act ? n_s : 1;
    ev.qv[k] = act ? n_s - 1 : 0;       // output points of the evaluation pass
    ev.mv[k] = act ? h.qv[k] + 1 : 1;   // input coefficients
    for (int i = 0; i < IGA_MAXM; ++i) sm.x[k][i] = act && i < n_s ? (double)i / (n_s - 1) : 0.0;
    for (int i = 0; i < (IGA_MAXQ + 1) * IGA_MAXM; ++i) ev.Pi1[k][i] = 0.0;
    if (!act) { ev.Pi1[k][0] = 1.0; continue; }
    nss *= n_s;
    const int q = h.qv[k];
    for (int sp = 0; sp < n_s; ++sp) {
      const double x = (double)sp / (n_s - 1);
      for (int c = 0; c <= q; ++c) {
        double b = 1.0;
        for (int r = 1; r <= c; ++r) b = b * (q - c + r) / r;
        ev.Pi1[k][sp * (q + 1) + c] = b * std::pow(x, c) * std::pow(1.0 - x, q - c);
      }
    }
  }
  sm.ns = nss;
  ev.ns = nss;
  const size_t smem = projection_error_smem_bytes(h.d, h.ns, n_s, h.npi);
  if (h.d == 2) {
    cudaError_t e = cudaFuncSetAttribute(kp_error<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    kp_error<2><<<(unsigned)h.n_tiles, 256, smem, s>>>(ic, sm, ev, ctrl, h.d_mknots, h.d_mspan, nu, e_tile, h.d_flag);
  } else {
    cudaError_t e = cudaFuncSetAttribute(kp_error<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    kp_error<3><<<(unsigned)h.n_tiles, 256, smem, s>>>(ic, sm, ev, ctrl, h.d_mknots, h.d_mspan, nu, e_tile, h.d_flag);
  }
  return cudaGetLastError();
}

template <int D>
__global__ void k5c_reduce(const __grid_constant__ InterpConst c_ip, const int *__restrict__ mspan, const double *__restrict__ gpart, int nact,
                           int64_t n_cp, double *__restrict__ grad) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_cp * D) return;
  int64_t k = idx / D;
  int a = (int)(idx % D);
  int ii[3] = {0, 0, 0};
  int64_t tmp = k;
  for (int kk = 0; kk < D; ++kk) { ii[kk] = (int)(tmp % c_ip.mn[kk]); tmp /= c_ip.mn[kk]; }
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  double acc = 0.0;
  const int mel2 = D > 2 ? c_ip.mel[2] : 1;
  for (int e2 = 0; e2 < mel2; ++e2) {
    int r2 = 0;
    if (D > 2) {
      int s = mspan[c_ip.soff[2] + e2];
      r2 = ii[2] - (s - c_ip.pm[2]);
      if (r2 < 0 || r2 > c_ip.pm[2]) continue;
    }
    for (int e1 = 0; e1 < c_ip.mel[1]; ++e1) {
      int s1 = mspan[c_ip.soff[1] + e1];
      int r1 = ii[1] - (s1 - c_ip.pm[1]);
      if (r1 < 0 || r1 > c_ip.pm[1]) continue;
      for (int e0 = 0; e0 < c_ip.mel[0]; ++e0) {
        int s0 = mspan[c_ip.soff[0] + e0];
        int r0 = ii[0] - (s0 - c_ip.pm[0]);
        if (r0 < 0 || r0 > c_ip.pm[0]) continue;
        const int64_t t = e0 + (int64_t)c_ip.mel[0] * (e1 + (int64_t)c_ip.mel[1] * e2) - c_ip.t_base;
        if (t < 0 || t >= c_ip.n_own) continue;   // tile of another shard (or this shard's halo)
        int ra = r0 + n1[0] * (r1 + n1[1] * r2);
        acc += gpart[((size_t)t * nact + ra) * D + a];
      }
    }
  }
  grad[idx] = acc;
}

template <int D, int Q>
static cudaError_t launch_k2(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                             double *coef, bool fm, cudaStream_t s) {
  if constexpr (Q >= 0 && K2Shape<D, (Q >= 0 ? Q : 0)>::REG) {
    if (h.iso && h.mv[0] == Q + 1) {   // interpolation: register path (else L2 projection, m > q+1)
      if (fm) {   // the K3 operand (sym layout)
        using S = K2Shape<D, Q, true>;
        const unsigned grid = (unsigned)((h.n_tiles + S::TPB - 1) / S::TPB);
        k2_interpolate<D, Q, true><<<grid, S::THREADS, 0, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan,
                                                               young, ypt, nu, coef, h.ks3, 4 * h.k3_split, h.tpc,
                                                               h.n_tiles, h.d_flag);
      } else {    // full coefficients, row-major (iga_interpolate)
        using S = K2Shape<D, Q, false>;
        const unsigned grid = (unsigned)((h.n_tiles + S::TPB - 1) / S::TPB);
        k2_interpolate<D, Q, false><<<grid, S::THREADS, 0, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan,
                                                                young, ypt, nu, coef, h.kstride, 0, h.tpc,
                                                                h.n_tiles, h.d_flag);
      }
      return cudaGetLastError();
    }
  }
  {
    const size_t sm = macro_smem_bytes(D, h.ns);
    cudaError_t e = cudaFuncSetAttribute(k2_interpolate_smem<D, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
    k2_interpolate_smem<D, Q><<<(unsigned)h.n_tiles, 256, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan,
                                                                   young, ypt, nu, coef, fm ? h.ks3 : h.kstride,
                                                                   (int)fm, 4 * h.k3_split, h.tpc, h.n_tiles,
                                                                   h.d_flag);
  }
  return cudaGetLastError();
}

template <int D, int Q>
static cudaError_t launch_k5b(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                              const double *W, double *gpart, cudaStream_t s) {
  if constexpr (Q >= 0 && K2Shape<D, (Q >= 0 ? Q : 0)>::REG) {
    if (h.iso && h.mv[0] == Q + 1) {   // interpolation (m = q+1): register path
      k5b_reverse_reg<D, Q><<<(unsigned)h.n_tiles_own, IGA_K5B_THREADS, 0, s>>>(
          make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young, ypt, nu, W, (int)h.k5_rows, h.tpc, h.k5_split,
          h.d_k5_gphys, gpart, h.d_flag);
      return cudaGetLastError();
    }
  }
  const size_t sm = k5b_smem_bytes(h, h.ns);
  cudaError_t e = cudaFuncSetAttribute(k5b_reverse<D, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e) return e;
  k5b_reverse<D, Q><<<(unsigned)h.n_tiles_own, IGA_K5B_THREADS, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young,
                                                        ypt, nu, W, (int)h.k5_rows, h.tpc, h.k5_split, h.k5_kap,
                                                        h.d_k5_gphys, gpart, h.d_flag);
  return cudaGetLastError();
}

// dispatch on (d, q): every index of the macro kernels is a compile-time constant;
// anisotropic degrees (Q = -1) take the runtime shared-memory path
#define IGA_DISPATCH_DQ(F, ...)                                                          \
  if (!h.iso) return h.d == 2 ? F<2, -1>(__VA_ARGS__) : F<3, -1>(__VA_ARGS__);           \
  switch (h.d * 10 + h.q) {                                                               \
    case 20: return F<2, 0>(__VA_ARGS__);                                                 \
    case 21: return F<2, 1>(__VA_ARGS__);                                                 \
    case 22: return F<2, 2>(__VA_ARGS__);                                                 \
    case 23: return F<2, 3>(__VA_ARGS__);                                                 \
    case 24: return F<2, 4>(__VA_ARGS__);                                                 \
    case 30: return F<3, 0>(__VA_ARGS__);                                                 \
    case 31: return F<3, 1>(__VA_ARGS__);                                                 \
    case 32: return F<3, 2>(__VA_ARGS__);                                                 \
    case 33: return F<3, 3>(__VA_ARGS__);                                                 \
    case 34: return F<3, 4>(__VA_ARGS__);                                                 \
    default: return cudaErrorInvalidValue;                                                \
  }

cudaError_t launch_interpolate(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                               double *coef, bool fm, cudaStream_t s) {
  IGA_DISPATCH_DQ(launch_k2, h, ctrl, young, ypt, nu, coef, fm, s)
}

cudaError_t launch_sens_reverse(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                                const double *W, double *gpart, cudaStream_t s) {
  IGA_DISPATCH_DQ(launch_k5b, h, ctrl, young, ypt, nu, W, gpart, s)
}

cudaError_t launch_sens_reduce(const Handle &h, const double *gpart, double *grad, cudaStream_t s) {
  int nact = 1;
  for (int k = 0; k < h.d; ++k) nact *= h.pm[k] + 1;
  int64_t n = h.n_cp * h.d;
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (h.d == 2)
    k5c_reduce<2><<<blocks, 256, 0, s>>>(make_interp_const(h), h.d_mspan, gpart, nact, h.n_cp, grad);
  else
    k5c_reduce<3><<<blocks, 256, 0, s>>>(make_interp_const(h), h.d_mspan, gpart, nact, h.n_cp, grad);
  return cudaGetLastError();
}

}  // namespace iga
