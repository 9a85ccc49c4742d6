// kernels_macro.cu — macro-scale kernels.
//
// K2 (interpolation, Eq. 42 in interpolation form, reading R1): per tile,
//   ∇F at the (q+1)^d tensor Gauss nodes of the element-local cube (Eq. 7 frame, R4),
//   Ā_ij[a,b] = D (λ ǧ_i[a] ǧ_j[b] + μ ǧ_j[a] ǧ_i[b] + μ (ǧ_i·ǧ_j) δ_ab)   (Eq. 37, App. A)
//   and the coefficients ⟨Ā⟩ = (V1⁻¹)^{⊗d} · samples (sum-factorised, one pass per direction).
//   HBM-bound: the only large traffic is the coefficient write (n_pi d⁴ doubles per tile).
//
// K5b (sensitivity, Eqs. 70-72): Ŵ_t = Πᵀ W_t, then at each node the analytic
//   reverse mode of S = ⟨Ŵ, Ā(J)⟩:
//     ∂S/∂J = S Gᵀ - Gᵀ Q Gᵀ,  G = J⁻¹,  Q = D(λ ∂T1/∂G + μ ∂T2/∂G + μ ∂T3/∂G)
//   chained to the macro control points through ∂J/∂P = h_β ∂_β N_k.
// K5c: deterministic reduction of the per-tile partials over the tiles sharing a
//   control point (fixed tile order, no atomics).
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
  for (int i = 0; i < (IGA_MAXQ + 1) * (IGA_MAXQ + 1); ++i) ic.Pi1[i] = h.Pi1[i];
  for (int i = 0; i <= IGA_MAXQ; ++i) ic.x[i] = h.interp_x[i];
  return ic;
}

// Shared per-tile macro data: 1D basis at the nodes and the active control points.
template <int D>
struct MacroTile {
  double B1[3][IGA_MAXQ + 1][IGA_MAXP + 1];
  double D1[3][IGA_MAXQ + 1][IGA_MAXP + 1];   // derivative w.r.t. ξ_k (includes span length)
  double P[(IGA_MAXP + 1) * (IGA_MAXP + 1) * (IGA_MAXP + 1) * 3];
  int nact;
};

template <int D>
__device__ void load_macro_tile(const InterpConst &c_ip, MacroTile<D> &mt, int64_t t, const double *__restrict__ ctrl,
                                const double *__restrict__ mknots, const int *__restrict__ mspan) {
  const int q = c_ip.q;
  int e[3] = {0, 0, 0};
  int64_t tmp = t;
  for (int k = 0; k < D; ++k) { e[k] = (int)(tmp % c_ip.mel[k]); tmp /= c_ip.mel[k]; }
  int tid = threadIdx.x;
  if (tid < D * (q + 1)) {
    int k = tid / (q + 1), m = tid % (q + 1);
    const double *U = mknots + c_ip.moff[k];
    int s = mspan[c_ip.soff[k] + e[k]];
    double h = U[s + 1] - U[s];
    double N[IGA_MAXP + 1], dN[IGA_MAXP + 1];
    bspline_eval(U, c_ip.pm[k], s, U[s] + h * c_ip.x[m], N, dN);
    for (int r = 0; r <= c_ip.pm[k]; ++r) {
      mt.B1[k][m][r] = N[r];
      mt.D1[k][m][r] = dN[r] * h;
    }
  }
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  int nact = n1[0] * n1[1] * n1[2];
  if (tid == 0) mt.nact = nact;
  for (int idx = tid; idx < nact * D; idx += blockDim.x) {
    int ra = idx / D, a = idx % D;
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    int64_t cp = 0;
    for (int k = D - 1; k >= 0; --k) {
      int s = mspan[c_ip.soff[k] + e[k]];
      cp = cp * c_ip.mn[k] + (s - c_ip.pm[k] + r[k]);
    }
    mt.P[idx] = ctrl[cp * D + a];
  }
}

// J[a][β] = ∂F_a/∂ξ_β at tensor node m (direction-0-fastest node index)
template <int D>
__device__ void macro_J(const InterpConst &c_ip, const MacroTile<D> &mt, int m, double J[D][D]) {
  const int q1 = c_ip.q + 1;
  int mm[3] = {m % q1, (m / q1) % q1, m / (q1 * q1)};
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  for (int a = 0; a < D; ++a)
    for (int b = 0; b < D; ++b) J[a][b] = 0.0;
  for (int ra = 0; ra < mt.nact; ++ra) {
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    double g[D];
    for (int be = 0; be < D; ++be) {
      double v = 1.0;
      for (int k = 0; k < D; ++k) v *= (k == be) ? mt.D1[k][mm[k]][r[k]] : mt.B1[k][mm[k]][r[k]];
      g[be] = v;
    }
    for (int a = 0; a < D; ++a) {
      double x = mt.P[ra * D + a];
      for (int be = 0; be < D; ++be) J[a][be] += x * g[be];
    }
  }
}

__device__ __forceinline__ void lame(double E, double nu, double &lam, double &mu) {
  lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  mu = E / (2.0 * (1.0 + nu));
}

// apply the 1D operator Op (row c, col m: out[c] = Σ_m Op[c][m] in[m], or its transpose)
// along direction `dir` of an (q+1)^D × ncomp array in shared memory.
template <int D>
__device__ void tensor_pass(const InterpConst &c_ip, const double *in, double *out, int dir, int ncomp, bool transpose) {
  const int q1 = c_ip.q + 1;
  int npi = 1;
  for (int k = 0; k < D; ++k) npi *= q1;
  int stride = 1;
  for (int k = 0; k < dir; ++k) stride *= q1;
  for (int idx = threadIdx.x; idx < npi * ncomp; idx += blockDim.x) {
    int C = idx / ncomp, comp = idx % ncomp;
    int c = (C / stride) % q1;
    int base = C - c * stride;
    double acc = 0.0;
    for (int m = 0; m < q1; ++m) {
      double op = transpose ? c_ip.Pi1[m * q1 + c] : c_ip.Pi1[c * q1 + m];
      acc += op * in[(base + m * stride) * ncomp + comp];
    }
    out[idx] = acc;
  }
}

template <int D>
__global__ void k2_interpolate(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
                               const int *__restrict__ mspan, const double *__restrict__ young, int ypt,
                               double nu, double *__restrict__ coef, int kstride, int fm, int *flag) {
  extern __shared__ double sm[];
  __shared__ MacroTile<D> mt;
  const int64_t t = blockIdx.x;
  const int q1 = c_ip.q + 1;
  int npi = 1;
  for (int k = 0; k < D; ++k) npi *= q1;
  constexpr int DD = D * D, NC = DD * DD;
  double *S0 = sm, *S1 = sm + npi * NC;
  load_macro_tile<D>(c_ip, mt, t, ctrl, mknots, mspan);
  __syncthreads();
  double E = young[ypt ? t : 0], lam, mu;
  lame(E, nu, lam, mu);
  for (int m = threadIdx.x; m < npi; m += blockDim.x) {
    double J[D][D], G[D][D];
    macro_J<D>(c_ip, mt, m, J);
    double det = det_inv<D>(J, G);
    if (!(det > 0.0)) raise_flag(flag, 2, (int)t, m);
    double gg[D][D];
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        double v = 0.0;
        for (int c = 0; c < D; ++c) v += G[i][c] * G[j][c];
        gg[i][j] = v;
      }
    double *o = S0 + m * NC;
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j)
        for (int a = 0; a < D; ++a)
          for (int b = 0; b < D; ++b)
            o[(i * D + j) * DD + a * D + b] =
                det * (lam * G[i][a] * G[j][b] + mu * G[j][a] * G[i][b] + (a == b ? mu * gg[i][j] : 0.0));
  }
  __syncthreads();
  double *in = S0, *out = S1;
  for (int dir = 0; dir < D; ++dir) {
    tensor_pass<D>(c_ip, in, out, dir, NC, false);
    __syncthreads();
    double *tmp = in; in = out; out = tmp;
  }
  // coefficient row n = t*DD + ab, column κ = ij*npi + C: row-major coef[n*kstride + κ]
  // (parity accessor) or the fragment-major K3 B operand (fm_index, BR = IGA_GEMM_BN)
  const int nk = DD * npi;
  for (int idx = threadIdx.x; idx < DD * nk; idx += blockDim.x) {
    int ab = idx / nk, kap = idx % nk;
    int ij = kap / npi, C = kap % npi;
    const int64_t n = t * DD + ab;
    const int64_t o = fm ? fm_index(n, kap, IGA_GEMM_BN, kstride / IGA_KCHUNK) : n * kstride + kap;
    coef[o] = in[C * NC + ij * DD + ab];
  }
}

template <int D>
__global__ void k5b_reverse(const __grid_constant__ InterpConst c_ip, const double *__restrict__ ctrl, const double *__restrict__ mknots,
                            const int *__restrict__ mspan, const double *__restrict__ young, int ypt, double nu,
                            const double *__restrict__ W, int kstride, double *__restrict__ gpart, int *flag) {
  extern __shared__ double sm[];
  __shared__ MacroTile<D> mt;
  const int64_t t = blockIdx.x;
  const int q1 = c_ip.q + 1;
  int npi = 1;
  for (int k = 0; k < D; ++k) npi *= q1;
  constexpr int DD = D * D, NC = DD * DD;
  double *S0 = sm, *S1 = sm + npi * NC, *dSdJ = sm + 2 * npi * NC;
  load_macro_tile<D>(c_ip, mt, t, ctrl, mknots, mspan);
  const int nk = DD * npi;
  const double *src = W + (size_t)t * DD * kstride;
  for (int idx = threadIdx.x; idx < DD * nk; idx += blockDim.x) {
    int ab = idx / nk, kap = idx % nk;
    int ij = kap / npi, C = kap % npi;
    S0[C * NC + ij * DD + ab] = src[(size_t)ab * kstride + kap];
  }
  __syncthreads();
  double *in = S0, *out = S1;
  for (int dir = 0; dir < D; ++dir) {   // Ŵ = Πᵀ W (transposed 1D operator per direction)
    tensor_pass<D>(c_ip, in, out, dir, NC, true);
    __syncthreads();
    double *tmp = in; in = out; out = tmp;
  }
  double E = young[ypt ? t : 0], lam, mu;
  lame(E, nu, lam, mu);
  for (int m = threadIdx.x; m < npi; m += blockDim.x) {
    const double *Wh = in + m * NC;   // Ŵ[ij*DD + ab]
    double J[D][D], G[D][D];
    macro_J<D>(c_ip, mt, m, J);
    double det = det_inv<D>(J, G);
    if (!(det > 0.0)) raise_flag(flag, 2, (int)t, m);
    double T1 = 0, T2 = 0, T3 = 0, w[D][D], gg[D][D];
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        double s = 0.0, v = 0.0;
        for (int a = 0; a < D; ++a) s += Wh[(i * D + j) * DD + a * D + a];
        for (int c = 0; c < D; ++c) v += G[i][c] * G[j][c];
        w[i][j] = s;
        gg[i][j] = v;
        T3 += s * v;
        for (int a = 0; a < D; ++a)
          for (int b = 0; b < D; ++b) {
            double x = Wh[(i * D + j) * DD + a * D + b];
            T1 += x * G[i][a] * G[j][b];
            T2 += x * G[j][a] * G[i][b];
          }
      }
    double S = det * (lam * T1 + mu * T2 + mu * T3);
    double Q[D][D];
    for (int mi = 0; mi < D; ++mi)
      for (int n = 0; n < D; ++n) {
        double d1 = 0, d2 = 0, d3 = 0;
        for (int j = 0; j < D; ++j)
          for (int b = 0; b < D; ++b) {
            d1 += Wh[(mi * D + j) * DD + n * D + b] * G[j][b];   // Σ_{j,b} Ŵ_{mj,nb} G_jb
            d1 += Wh[(j * D + mi) * DD + b * D + n] * G[j][b];   // Σ_{i,a} Ŵ_{im,an} G_ia
            d2 += Wh[(j * D + mi) * DD + n * D + b] * G[j][b];   // Σ_{i,b} Ŵ_{im,nb} G_ib
            d2 += Wh[(mi * D + j) * DD + b * D + n] * G[j][b];   // Σ_{j,a} Ŵ_{mj,an} G_ja
          }
        for (int j = 0; j < D; ++j) d3 += (w[mi][j] + w[j][mi]) * G[j][n];
        Q[mi][n] = det * (lam * d1 + mu * d2 + mu * d3);
      }
    // ∂S/∂J[a][β] = S G[β][a] - Σ_{i,n} G[i][a] Q[i][n] G[β][n]
    double *o = dSdJ + m * DD;
    for (int a = 0; a < D; ++a)
      for (int be = 0; be < D; ++be) {
        double v = S * G[be][a];
        for (int i = 0; i < D; ++i)
          for (int n = 0; n < D; ++n) v -= G[i][a] * Q[i][n] * G[be][n];
        o[a * D + be] = v;
      }
  }
  __syncthreads();
  // chain to the active control points: g[r][a] = Σ_m Σ_β ∂S/∂J[a][β] ∂_β N_r(ξ_m)
  int n1[3] = {c_ip.pm[0] + 1, D > 1 ? c_ip.pm[1] + 1 : 1, D > 2 ? c_ip.pm[2] + 1 : 1};
  for (int idx = threadIdx.x; idx < mt.nact * D; idx += blockDim.x) {
    int ra = idx / D, a = idx % D;
    int r[3] = {ra % n1[0], (ra / n1[0]) % n1[1], ra / (n1[0] * n1[1])};
    double acc = 0.0;
    for (int m = 0; m < npi; ++m) {
      int mm[3] = {m % q1, (m / q1) % q1, m / (q1 * q1)};
      for (int be = 0; be < D; ++be) {
        double v = 1.0;
        for (int k = 0; k < D; ++k) v *= (k == be) ? mt.D1[k][mm[k]][r[k]] : mt.B1[k][mm[k]][r[k]];
        acc += dSdJ[m * DD + a * D + be] * v;
      }
    }
    gpart[((size_t)t * mt.nact + ra) * D + a] = acc;
  }
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
        int64_t t = e0 + (int64_t)c_ip.mel[0] * (e1 + (int64_t)c_ip.mel[1] * e2);
        int ra = r0 + n1[0] * (r1 + n1[1] * r2);
        acc += gpart[((size_t)t * nact + ra) * D + a];
      }
    }
  }
  grad[idx] = acc;
}

static size_t macro_smem(const Handle &h, int extra_per_node) {
  int npi = h.npi, dd = h.d * h.d;
  return sizeof(double) * ((size_t)2 * npi * dd * dd + (size_t)npi * extra_per_node);
}

cudaError_t launch_interpolate(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                               double *coef, bool fm, cudaStream_t s) {
  size_t sm = macro_smem(h, 0);
  if (h.d == 2) {
    cudaFuncSetAttribute(k2_interpolate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k2_interpolate<2><<<(unsigned)h.n_tiles, 128, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young, ypt, nu, coef, h.kstride, (int)fm, h.d_flag);
  } else {
    cudaFuncSetAttribute(k2_interpolate<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k2_interpolate<3><<<(unsigned)h.n_tiles, 128, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young, ypt, nu, coef, h.kstride, (int)fm, h.d_flag);
  }
  return cudaGetLastError();
}

cudaError_t launch_sens_reverse(const Handle &h, const double *ctrl, const double *young, int ypt, double nu,
                                const double *W, double *gpart, cudaStream_t s) {
  size_t sm = macro_smem(h, h.d * h.d);
  if (h.d == 2) {
    cudaFuncSetAttribute(k5b_reverse<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k5b_reverse<2><<<(unsigned)h.n_tiles, 128, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young, ypt, nu, W, h.kstride, gpart, h.d_flag);
  } else {
    cudaFuncSetAttribute(k5b_reverse<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k5b_reverse<3><<<(unsigned)h.n_tiles, 128, sm, s>>>(make_interp_const(h), ctrl, h.d_mknots, h.d_mspan, young, ypt, nu, W, h.kstride, gpart, h.d_flag);
  }
  return cudaGetLastError();
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
