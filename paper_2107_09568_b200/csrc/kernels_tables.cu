// kernels_tables.cu — K1: lookup tables 𝔎_p by micro-scale Gauss quadrature
// (Eqs. 51-52; matricised per Eq. 57).
//
//   𝔎_p[(A,B)][κ=(i*d+j)*n_pi + C] = Σ_spans Σ_g w_g |span| det J_T
//                                     (J_T⁻ᵀ∇_θR_A)_i (J_T⁻ᵀ∇_θR_B)_j N_C(𝒯(θ_g))
//
// Two kernels: (a) one thread per tile quadrature point evaluates the point data
// (w·det J_T, ξ-gradients of the (p+1)^d active functions, N_C at ξ = 𝒯(θ));
// (b) one CTA per table row (A,B) owns all κ entries of that row and sums over the
// spans shared by A and B in a fixed order (deterministic, no atomics).
// Offline per the paper; timed separately from the metric.
#include "device_common.cuh"

namespace iga {

__constant__ DevPatch c_patches[64];
__constant__ double c_gx[16], c_gw[16];

template <int D>
__global__ void k1_point_data(int n_patches, int n_g, int p, int3 qv, const double *__restrict__ tile_ctrl,
                              const double *__restrict__ knots, const int *__restrict__ elspan, int total_pts,
                              double *__restrict__ wD, double *__restrict__ G, double *__restrict__ Nc,
                              double *__restrict__ Rv, int *flag) {
  int gp = blockIdx.x * blockDim.x + threadIdx.x;
  if (gp >= total_pts) return;
  int pi = 0;
  while (pi + 1 < n_patches && gp >= c_patches[pi + 1].pt_off) ++pi;
  const DevPatch &P = c_patches[pi];
  int ng_d = 1;
  for (int k = 0; k < D; ++k) ng_d *= n_g;
  int local = gp - P.pt_off;
  int span_lin = local / ng_d, g = local % ng_d;
  int e[3], gi[3], s[3];
  for (int k = 0, sl = span_lin, gg = g; k < D; ++k) {
    e[k] = sl % P.n_span[k];
    sl /= P.n_span[k];
    gi[k] = gg % n_g;
    gg /= n_g;
  }
  double N1[3][IGA_MAXP + 1], D1[3][IGA_MAXP + 1], w = 1.0;
  for (int k = 0; k < D; ++k) {
    const double *U = knots + P.knot_off[k];
    s[k] = elspan[P.elspan_off[k] + e[k]];
    double h = U[s[k] + 1] - U[s[k]];
    double th = U[s[k]] + h * c_gx[gi[k]];
    w *= c_gw[gi[k]] * h;
    bspline_eval(U, p, s[k], th, N1[k], D1[k]);
  }
  const int n1 = p + 1;
  int nact = 1;
  for (int k = 0; k < D; ++k) nact *= n1;
  // ξ = 𝒯(θ), J_T[a][k] = ∂ξ_a/∂θ_k
  double xi[D], JT[D][D];
  for (int a = 0; a < D; ++a) {
    xi[a] = 0.0;
    for (int k = 0; k < D; ++k) JT[a][k] = 0.0;
  }
  for (int la = 0; la < nact; ++la) {
    int r[3] = {la % n1, (la / n1) % n1, la / (n1 * n1)};
    int ii[3];
    for (int k = 0; k < D; ++k) ii[k] = s[k] - p + r[k];
    int A = ii[0] + P.n[0] * (ii[1] + (D == 3 ? P.n[1] * ii[2] : 0));
    const double *x = tile_ctrl + (size_t)(P.ctrl_off + A) * D;
    double R = 1.0, dR[D];
    for (int k = 0; k < D; ++k) R *= N1[k][r[k]];
    for (int m = 0; m < D; ++m) {
      double v = 1.0;
      for (int k = 0; k < D; ++k) v *= (k == m) ? D1[k][r[k]] : N1[k][r[k]];
      dR[m] = v;
    }
    for (int a = 0; a < D; ++a) {
      xi[a] += R * x[a];
      for (int m = 0; m < D; ++m) JT[a][m] += dR[m] * x[a];
    }
  }
  double Ginv[D][D];
  double det = det_inv<D>(JT, Ginv);   // Ginv[m][a] = (J_T⁻¹)[m][a] = ∂θ_m/∂ξ_a
  if (!(det > 0.0)) raise_flag(flag, 1, pi, gp);
  wD[gp] = w * det;
  double *Gp = G + (size_t)gp * nact * D;
  for (int la = 0; la < nact; ++la) {
    int r[3] = {la % n1, (la / n1) % n1, la / (n1 * n1)};
    double R = 1.0;
    for (int k = 0; k < D; ++k) R *= N1[k][r[k]];
    Rv[(size_t)gp * nact + la] = R;
    double dR[D];
    for (int m = 0; m < D; ++m) {
      double v = 1.0;
      for (int k = 0; k < D; ++k) v *= (k == m) ? D1[k][r[k]] : N1[k][r[k]];
      dR[m] = v;
    }
    for (int a = 0; a < D; ++a) {
      double v = 0.0;
      for (int m = 0; m < D; ++m) v += Ginv[m][a] * dR[m];   // (J_T⁻ᵀ ∇_θ R)_a
      Gp[la * D + a] = v;
    }
  }
  // N_C(ξ) = Π_k B_{c_k}^{q_k}(ξ_k) with per-direction degrees (anisotropic Q)
  const int q[3] = {qv.x, qv.y, qv.z};
  int npi = 1;
  for (int k = 0; k < D; ++k) npi *= q[k] + 1;
  double B1[3][IGA_MAXQ + 1];
  for (int k = 0; k < D; ++k)
    for (int c = 0; c <= q[k]; ++c) B1[k][c] = bernstein1(q[k], c, xi[k]);
  double *Np = Nc + (size_t)gp * npi;
  for (int C = 0; C < npi; ++C) {
    int c[3] = {C % (q[0] + 1), (C / (q[0] + 1)) % (q[1] + 1), C / ((q[0] + 1) * (q[1] + 1))};
    double v = 1.0;
    for (int k = 0; k < D; ++k) v *= B1[k][c[k]];
    Np[C] = v;
  }
}

template <int D>
__global__ void k1_table_rows(int n_patches, int n_g, int p, int npi, int nk, int kstride, int64_t M, int64_t ldT,
                              const int *__restrict__ row_patch, const int *__restrict__ pairA,
                              const int *__restrict__ pairB, const int *__restrict__ elspan,
                              const double *__restrict__ wD, const double *__restrict__ G,
                              const double *__restrict__ Nc, double *__restrict__ table) {
  int64_t row = blockIdx.x;
  int pi = row_patch[row];
  const DevPatch &P = c_patches[pi];
  int A = pairA[row] - P.ctrl_off, B = pairB[row] - P.ctrl_off;
  int a[3] = {A % P.n[0], (A / P.n[0]) % P.n[1], A / (P.n[0] * P.n[1])};
  int b[3] = {B % P.n[0], (B / P.n[0]) % P.n[1], B / (P.n[0] * P.n[1])};
  const int n1 = p + 1;
  int nact = 1, ng_d = 1;
  for (int k = 0; k < D; ++k) { nact *= n1; ng_d *= n_g; }
  // element ranges per direction where both functions are nonzero: knot span s in
  // [max(a,b), min(a,b)+p]
  int elo[3], ehi[3];
  for (int k = 0; k < 3; ++k) { elo[k] = 0; ehi[k] = 0; }
  for (int k = 0; k < D; ++k) {
    int slo = max(a[k], b[k]), shi = min(a[k], b[k]) + p;
    const int *es = elspan + P.elspan_off[k];
    elo[k] = P.n_span[k];
    ehi[k] = -1;
    for (int e = 0; e < P.n_span[k]; ++e)
      if (es[e] >= slo && es[e] <= shi) { elo[k] = min(elo[k], e); ehi[k] = max(ehi[k], e); }
  }
  for (int kap = threadIdx.x; kap < nk; kap += blockDim.x) {
    int i = kap / (D * npi), j = (kap / npi) % D, C = kap % npi;
    double acc = 0.0;
    for (int e2 = (D == 3 ? elo[2] : 0); e2 <= (D == 3 ? ehi[2] : 0); ++e2)
      for (int e1 = elo[1]; e1 <= ehi[1]; ++e1)
        for (int e0 = elo[0]; e0 <= ehi[0]; ++e0) {
          int e[3] = {e0, e1, e2};
          int span_lin = e0 + P.n_span[0] * (e1 + P.n_span[1] * e2);
          int la = 0, lb = 0;
          for (int k = D - 1; k >= 0; --k) {
            int s = elspan[P.elspan_off[k] + e[k]];
            la = la * n1 + (a[k] - (s - p));
            lb = lb * n1 + (b[k] - (s - p));
          }
          int64_t base = P.pt_off + (int64_t)span_lin * ng_d;
          for (int g = 0; g < ng_d; ++g) {
            int64_t pt = base + g;
            const double *Gp = G + (size_t)pt * nact * D;
            acc += wD[pt] * Gp[la * D + i] * Gp[lb * D + j] * Nc[(size_t)pt * npi + C];
          }
        }
    table[row * kstride + kap] = acc;
  }
}

// Load / volume tables (Eq. 53 body part, Eq. 18), offline:
//   𝔉[A][C] = Σ_spans(A) Σ_g w_g |span| det J_T R_A N_C(𝒯(θ_g))   one CTA per control point
//   t^h[C]  = Σ_patches Σ_spans Σ_g w_g |span| det J_T N_C(𝒯(θ_g))  one thread per C
template <int D>
__global__ void k1_load_rows(int n_patches, int n_g, int p, int npi, const int *__restrict__ elspan,
                             const double *__restrict__ wD, const double *__restrict__ Nc,
                             const double *__restrict__ Rv, double *__restrict__ F) {
  const int Aglob = blockIdx.x;
  int pi = 0;
  while (pi + 1 < n_patches && Aglob >= c_patches[pi + 1].ctrl_off) ++pi;
  const DevPatch &P = c_patches[pi];
  const int A = Aglob - P.ctrl_off;
  const int a[3] = {A % P.n[0], (A / P.n[0]) % P.n[1], A / (P.n[0] * P.n[1])};
  const int n1 = p + 1;
  int nact = 1, ng_d = 1;
  for (int k = 0; k < D; ++k) { nact *= n1; ng_d *= n_g; }
  int elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
  for (int k = 0; k < D; ++k) {   // elements whose span s satisfies a_k <= s <= a_k + p
    const int *es = elspan + P.elspan_off[k];
    elo[k] = P.n_span[k];
    ehi[k] = -1;
    for (int e = 0; e < P.n_span[k]; ++e)
      if (es[e] >= a[k] && es[e] <= a[k] + p) { elo[k] = min(elo[k], e); ehi[k] = max(ehi[k], e); }
  }
  for (int C = threadIdx.x; C < npi; C += blockDim.x) {
    double acc = 0.0;
    for (int e2 = (D == 3 ? elo[2] : 0); e2 <= (D == 3 ? ehi[2] : 0); ++e2)
      for (int e1 = elo[1]; e1 <= ehi[1]; ++e1)
        for (int e0 = elo[0]; e0 <= ehi[0]; ++e0) {
          const int e[3] = {e0, e1, e2};
          const int span_lin = e0 + P.n_span[0] * (e1 + P.n_span[1] * e2);
          int la = 0;
          for (int k = D - 1; k >= 0; --k) la = la * n1 + (a[k] - (elspan[P.elspan_off[k] + e[k]] - p));
          const int64_t base = P.pt_off + (int64_t)span_lin * ng_d;
          for (int g = 0; g < ng_d; ++g) {
            const int64_t pt = base + g;
            acc += wD[pt] * Rv[(size_t)pt * nact + la] * Nc[(size_t)pt * npi + C];
          }
        }
    F[(size_t)Aglob * npi + C] = acc;
  }
}

__global__ void k1_volume_table(int total_pts, int npi, const double *__restrict__ wD, const double *__restrict__ Nc,
                                double *__restrict__ th) {
  const int C = blockIdx.x * blockDim.x + threadIdx.x;
  if (C >= npi) return;
  double acc = 0.0;
  for (int pt = 0; pt < total_pts; ++pt) acc += wD[pt] * Nc[(size_t)pt * npi + C];
  th[C] = acc;
}

// Offline re-layout of the row-major table into the two fragment-major GEMM operands
// (device_common.cuh fm_index) of the Eq. 38-reduced contraction: K3's A
// (rows = table rows, BR = IGA_K3_BM; columns part 1 = [T_ii | T_ij + T_ji] per P1 pair and
// C, part 2 = [T_ij − T_ji] per P2 pair and C starting at k1) and K5a's A (the same
// quantities as rows κ, part 2 from k5s; reduction columns = table rows with each patch
// padded to 16, BR = IGA_K5_BM).
template <int D>
__global__ void k1_pack(const double *__restrict__ table, int64_t M, int npi, int kstride,
                        const int32_t *__restrict__ k5_col, double *__restrict__ tabA, int nkcA, int k1,
                        double *__restrict__ tabAT, int brT, int nkcT, int k5s, const int32_t *__restrict__ gphys) {
  constexpr int NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2;
  const int ns = (NP1 + NP2) * npi;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= M * ns) return;
  const int64_t r = idx / ns;
  const int sk = (int)(idx % ns), p = sk / npi, C = sk % npi;
  const double *T = table + r * kstride;
  int i, j, kA, kT;
  double v;
  if (p < NP1) {
    sym_pair(D, p, i, j);
    v = i == j ? T[(i * D + i) * npi + C] : T[(i * D + j) * npi + C] + T[(j * D + i) * npi + C];
    kA = kT = sk;
  } else {
    anti_pair(D, p - NP1, i, j);
    v = T[(i * D + j) * npi + C] - T[(j * D + i) * npi + C];
    kA = k1 + (sk - NP1 * npi);
    kT = k5s + (sk - NP1 * npi);
  }
  tabA[fm_index(r, kA, IGA_K3_BM, nkcA)] = v;
  tabAT[fm_index(gphys[kT >> 3] * 8 + (kT & 7), k5_col[r], brT, nkcT)] = v;   // balanced κ placement
}

cudaError_t launch_pack_tables(const Handle &h, cudaStream_t s) {
  const int64_t n = h.M * (h.n_p1 + h.n_p2) * h.npi;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (h.d == 2)
    k1_pack<2><<<blocks, 256, 0, s>>>(h.d_table, h.M, h.npi, h.kstride, h.d_k5_col, h.d_tabA, h.ks3 / IGA_KCHUNK,
                                      4 * h.k3_split, h.d_tabAT, IGA_K5_BM, (int)(h.Kp / IGA_KCHUNK), h.k5_split,
                                      h.d_k5_gphys);
  else
    k1_pack<3><<<blocks, 256, 0, s>>>(h.d_table, h.M, h.npi, h.kstride, h.d_k5_col, h.d_tabA, h.ks3 / IGA_KCHUNK,
                                      4 * h.k3_split, h.d_tabAT, IGA_K5_BM, (int)(h.Kp / IGA_KCHUNK), h.k5_split,
                                      h.d_k5_gphys);
  return cudaGetLastError();
}

cudaError_t launch_tables(const Handle &h, const DevPatch *dpatches, int n_patches, const double *d_tile_ctrl,
                          const double *d_tile_knots, const int *d_tile_elspan, const double *gx,
                          const double *gw, int total_pts, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemcpyToSymbolAsync(c_patches, dpatches, sizeof(DevPatch) * n_patches, 0, cudaMemcpyHostToDevice, s))) return e;
  if ((e = cudaMemcpyToSymbolAsync(c_gx, gx, sizeof(double) * h.n_g, 0, cudaMemcpyHostToDevice, s))) return e;
  if ((e = cudaMemcpyToSymbolAsync(c_gw, gw, sizeof(double) * h.n_g, 0, cudaMemcpyHostToDevice, s))) return e;
  int nact = 1;
  for (int k = 0; k < h.d; ++k) nact *= (h.p + 1);
  double *wD, *G, *Nc, *Rv;
  int *row_patch;
  if ((e = cudaMallocAsync((void **)&Rv, sizeof(double) * (size_t)total_pts * nact, s))) return e;
  if ((e = cudaMallocAsync((void **)&wD, sizeof(double) * total_pts, s))) return e;
  if ((e = cudaMallocAsync((void **)&G, sizeof(double) * (size_t)total_pts * nact * h.d, s))) return e;
  if ((e = cudaMallocAsync((void **)&Nc, sizeof(double) * (size_t)total_pts * h.npi, s))) return e;
  if ((e = cudaMallocAsync((void **)&row_patch, sizeof(int) * h.M, s))) return e;
  std::vector<int> rp(h.M);
  for (int pi = 0; pi < n_patches; ++pi)
    for (int r = 0; r < h.patches[pi].n_nz; ++r) rp[h.patches[pi].row_off + r] = pi;
  if ((e = cudaMemcpyAsync(row_patch, rp.data(), sizeof(int) * h.M, cudaMemcpyHostToDevice, s))) return e;
  int threads = 128, blocks = (total_pts + threads - 1) / threads;
  if (h.d == 2)
    k1_point_data<2><<<blocks, threads, 0, s>>>(n_patches, h.n_g, h.p, make_int3(h.qv[0], h.qv[1], h.qv[2]), d_tile_ctrl, d_tile_knots, d_tile_elspan,
                                                total_pts, wD, G, Nc, Rv, h.d_flag);
  else
    k1_point_data<3><<<blocks, threads, 0, s>>>(n_patches, h.n_g, h.p, make_int3(h.qv[0], h.qv[1], h.qv[2]), d_tile_ctrl, d_tile_knots, d_tile_elspan,
                                                total_pts, wD, G, Nc, Rv, h.d_flag);
  if ((e = cudaGetLastError())) return e;
  int tpb = h.nk >= 256 ? 256 : 128;
  if (h.d == 2)
    k1_table_rows<2><<<(unsigned)h.M, tpb, 0, s>>>(n_patches, h.n_g, h.p, h.npi, h.nk, h.kstride, h.M, (h.M + IGA_KCHUNK - 1) / IGA_KCHUNK * IGA_KCHUNK, row_patch,
                                                   h.d_pairA, h.d_pairB, d_tile_elspan, wD, G, Nc, h.d_table);
  else
    k1_table_rows<3><<<(unsigned)h.M, tpb, 0, s>>>(n_patches, h.n_g, h.p, h.npi, h.nk, h.kstride, h.M, (h.M + IGA_KCHUNK - 1) / IGA_KCHUNK * IGA_KCHUNK, row_patch,
                                                   h.d_pairA, h.d_pairB, d_tile_elspan, wD, G, Nc, h.d_table);
  if ((e = cudaGetLastError())) return e;
  if (h.d == 2)
    k1_load_rows<2><<<(unsigned)h.n_local_ctrl, 64, 0, s>>>(n_patches, h.n_g, h.p, h.npi, d_tile_elspan, wD, Nc, Rv, h.d_F);
  else
    k1_load_rows<3><<<(unsigned)h.n_local_ctrl, 64, 0, s>>>(n_patches, h.n_g, h.p, h.npi, d_tile_elspan, wD, Nc, Rv, h.d_F);
  k1_volume_table<<<(h.npi + 63) / 64, 64, 0, s>>>(total_pts, h.npi, wD, Nc, h.d_th);
  if ((e = cudaGetLastError())) return e;
  cudaFreeAsync(Rv, s);
  cudaFreeAsync(wD, s);
  cudaFreeAsync(G, s);
  cudaFreeAsync(Nc, s);
  cudaFreeAsync(row_patch, s);
  return cudaSuccess;
}

}  // namespace iga
