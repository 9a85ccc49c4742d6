// kernels_scatter.cu — K4: local element blocks -> full symmetric CSR values
// ("any scientific library ... sparse matrix data structures", §3.2.4
// step 4 P:425; reading R9 for the symmetric storage).
//
// Owner computes, atomic-free and deterministic: one warp per global node row I.
// Lane j owns block (I, J_j) of the block row; its contributor list (tile, local row,
// transposed?) was built once on the host, sorted by (tile, row).  Each contributor is
// a 9-double (3D) contiguous block of `local`; diagonal pairs (A = B) contribute their
// upper triangle to both triangles so K is bitwise symmetric.  The node's d scalar
// rows are one contiguous segment of the CSR value array: lane j writes d×d values at
// row_base + a*d*nnzb + d*j + b.
#include "device_common.cuh"

namespace iga {

template <int D>
__global__ void __launch_bounds__(256)
k4_scatter(const double *__restrict__ local, double *__restrict__ vals, const int64_t *__restrict__ brow_ptr,
           const uint8_t *__restrict__ bcnt, const int64_t *__restrict__ cstart,
           const uint32_t *__restrict__ contrib, const int *__restrict__ pairA, const int *__restrict__ pairB,
           int64_t n_nodes, int64_t ldl, int rb) {
  constexpr int DD = D * D;
  const int lane = threadIdx.x & 31;
  const int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (I >= n_nodes) return;
  const int64_t b0 = brow_ptr[I];
  const int nb = (int)(brow_ptr[I + 1] - b0);
  const int64_t rowbase = DD * b0, rowlen = (int64_t)D * nb;
  int64_t cbase = cstart[I];
  const uint32_t rmask = (1u << rb) - 1u;
  for (int jb0 = 0; jb0 < nb; jb0 += 32) {
    const int jb = jb0 + lane;
    const int cnt = jb < nb ? bcnt[b0 + jb] : 0;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t c0 = cbase + incl - cnt;
    double acc[DD];
#pragma unroll
    for (int e = 0; e < DD; ++e) acc[e] = 0.0;
    for (int k = 0; k < cnt; ++k) {
      const uint32_t pk = contrib[c0 + k];
      const int64_t t = pk >> (rb + 1);
      const int r = (int)((pk >> 1) & rmask);
      const double *L = local + (int64_t)r * ldl + t * DD;
      double l[DD];
#pragma unroll
      for (int e = 0; e < DD; ++e) l[e] = L[e];
      if (pairA[r] == pairB[r]) {
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) acc[a * D + b] += a <= b ? l[a * D + b] : l[b * D + a];
      } else if (pk & 1u) {
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) acc[a * D + b] += l[b * D + a];
      } else {
#pragma unroll
        for (int e = 0; e < DD; ++e) acc[e] += l[e];
      }
    }
    if (jb < nb) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) vals[rowbase + a * rowlen + (int64_t)D * jb + b] = acc[a * D + b];
    }
    cbase += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// row_ptr / col_idx of the scalar CSR from the block CSR (interleaved DOFs, R9).
template <int D>
__global__ void k4_expand_pattern(const int64_t *__restrict__ brow_ptr, const int32_t *__restrict__ bcol,
                                  int64_t n_nodes, int64_t *__restrict__ row_ptr, int32_t *__restrict__ col_idx) {
  constexpr int DD = D * D;
  const int lane = threadIdx.x & 31;
  const int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (I >= n_nodes) return;
  const int64_t b0 = brow_ptr[I];
  const int nb = (int)(brow_ptr[I + 1] - b0);
  const int64_t rowbase = DD * b0, rowlen = (int64_t)D * nb;
  if (lane < D) row_ptr[I * D + lane] = rowbase + lane * rowlen;
  if (I == n_nodes - 1 && lane == 0) row_ptr[n_nodes * D] = DD * brow_ptr[n_nodes];
  for (int jb = lane; jb < nb; jb += 32) {
    int32_t J = bcol[b0 + jb];
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) col_idx[rowbase + a * rowlen + (int64_t)D * jb + b] = J * D + b;
  }
}

cudaError_t launch_scatter(const Handle &h, const double *local, double *vals, cudaStream_t s) {
  int64_t threads = h.n_nodes * 32;
  unsigned blocks = (unsigned)((threads + 255) / 256);
  int64_t ldl = h.n_tiles * h.d * h.d;
  if (h.d == 2)
    k4_scatter<2><<<blocks, 256, 0, s>>>(local, vals, h.d_brow_ptr, h.d_bcnt, h.d_cstart, h.d_contrib, h.d_pairA,
                                         h.d_pairB, h.n_nodes, ldl, h.row_bits);
  else
    k4_scatter<3><<<blocks, 256, 0, s>>>(local, vals, h.d_brow_ptr, h.d_bcnt, h.d_cstart, h.d_contrib, h.d_pairA,
                                         h.d_pairB, h.n_nodes, ldl, h.row_bits);
  return cudaGetLastError();
}

cudaError_t launch_expand_pattern(const Handle &h, cudaStream_t s) {
  int64_t threads = h.n_nodes * 32;
  unsigned blocks = (unsigned)((threads + 255) / 256);
  if (h.d == 2)
    k4_expand_pattern<2><<<blocks, 256, 0, s>>>(h.d_brow_ptr, h.d_bcol, h.n_nodes, h.d_row_ptr, h.d_col_idx);
  else
    k4_expand_pattern<3><<<blocks, 256, 0, s>>>(h.d_brow_ptr, h.d_bcol, h.n_nodes, h.d_row_ptr, h.d_col_idx);
  return cudaGetLastError();
}

}  // namespace iga
