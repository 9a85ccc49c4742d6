// kernels_scatter.cu — K4: the blocks of K that several (tile, local row) contributions
// share ("any scientific library ... sparse matrix data structures",
// §3.2.4 step 4 P:425; reading R9 for the symmetric storage).
//
// Single-contribution blocks are written by the K3 epilogue directly.  A block with
// several contributions — control points on tile faces shared by neighbouring tiles,
// or on declared patch interfaces inside a tile — receives one side slot per
// contribution from K3; here its slots are summed in the fixed order built on the host
// (sorted by (tile, row)), transposing the slots recorded in the (J,I) orientation, and
// K(I,J) and K(J,I) = K(I,J)ᵀ are written.  Diagonal blocks take the upper triangle for
// both triangles.  No atomics; bitwise deterministic.
#include "device_common.cuh"

namespace iga {

// sum of the slots of multi block m (fixed slot order; slots recorded in the (J,I)
// orientation transposed)
template <int D>
__device__ __forceinline__ void k4_sum(const double *__restrict__ side, const int32_t *__restrict__ mslot0,
                                       const uint8_t *__restrict__ slot_tr, int64_t m, double *acc) {
  constexpr int DD = D * D;
  const int s0 = mslot0[m], s1 = mslot0[m + 1];
#pragma unroll
  for (int e = 0; e < DD; ++e) acc[e] = 0.0;
  for (int sl = s0; sl < s1; sl += 2) {   // two slots per iteration, loads first
    const bool two = sl + 1 < s1;
    const double *L0 = side + (int64_t)sl * DD, *L1 = side + (int64_t)(two ? sl + 1 : sl) * DD;
    double l0[DD], l1[DD];
#pragma unroll
    for (int e = 0; e < DD; ++e) { l0[e] = L0[e]; l1[e] = L1[e]; }
    const bool t0 = slot_tr[sl], t1 = two && slot_tr[sl + 1];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) acc[a * D + b] += t0 ? l0[b * D + a] : l0[a * D + b];
    if (two) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) acc[a * D + b] += t1 ? l1[b * D + a] : l1[a * D + b];
    }
  }
}

// Thread m: pass 1 writes K(I,J) of multi block m (blocks ordered by (I, J)); pass 2 writes
// K(J,I) of block mperm[m] (ordered by (J, I)).  Both orders put neighbouring blocks of one
// CSR row in neighbouring lanes; the d-double row segments are stored warp-cooperatively
// from a shared-memory copy of the sums (whole sectors for runs of adjacent blocks).
template <int D>
__global__ void __launch_bounds__(256)
k4_multi(const double *__restrict__ side, const MultiBlock *__restrict__ mblk, const int32_t *__restrict__ mslot0,
         const uint8_t *__restrict__ slot_tr, const int32_t *__restrict__ mperm, int64_t n_multi,
         double *__restrict__ vals) {
  constexpr int DD = D * D;
  __shared__ double sacc[2][256 * DD];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + tid;
  const bool live = m < n_multi;
  const int64_t mt = live ? mperm[m] : 0;
  MultiBlock b1{}, b2{};
  double acc1[DD], acc2[DD];
  if (live) {
    b1 = mblk[m];
    b2 = mblk[mt];
    k4_sum<D>(side, mslot0, slot_tr, m, acc1);
    k4_sum<D>(side, mslot0, slot_tr, mt, acc2);
  }
#pragma unroll
  for (int e = 0; e < DD; ++e) {
    sacc[0][tid * DD + e] = live ? acc1[e] : 0.0;
    sacc[1][tid * DD + e] = live ? acc2[e] : 0.0;
  }
  __syncwarp();
  const int wbase = tid & ~31;
  // lanes hold (o = CSR offset of their block's first row segment or -1, row stride,
  // diagonal?); word w of the warp's row segments comes from lane w/D, column w%D, and the
  // D row segments of a block are o, o + stride, ...: one set of shuffles per block
  auto coop = [&](int64_t o, int str, bool dg, int pass) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int w = 32 * j + lane, src = w / D, c = w - src * D;
      const int64_t ob = __shfl_sync(0xffffffffu, o, src);
      const int sstr = __shfl_sync(0xffffffffu, str, src);
      const bool db = __shfl_sync(0xffffffffu, (int)dg, src) != 0;
      if (ob >= 0) {
#pragma unroll
        for (int idx = 0; idx < D; ++idx) {
          int ra = pass ? c : idx, cb = pass ? idx : c;
          if (db && ra > cb) { const int x = ra; ra = cb; cb = x; }
          vals[ob + (int64_t)idx * sstr + c] = sacc[pass][(wbase + src) * DD + ra * D + cb];
        }
      }
    }
  };
  const bool dg1 = b1.off_ij == b1.off_ji;
  coop(live ? b1.off_ij : -1, b1.stride_i, dg1, 0);
  // diagonal blocks are complete after pass 1; off_ji < 0: row J belongs to another shard
  const bool w2 = live && b2.off_ji >= 0 && b2.off_ij != b2.off_ji;
  coop(w2 ? b2.off_ji : -1, b2.stride_j, false, 1);
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

cudaError_t launch_scatter_multi(const Handle &h, double *vals, cudaStream_t s) {
  if (h.n_multi == 0) return cudaSuccess;
  unsigned blocks = (unsigned)((h.n_multi + 255) / 256);
  if (h.d == 2)
    k4_multi<2><<<blocks, 256, 0, s>>>(h.d_side, h.d_mblk, h.d_mslot0, h.d_slot_tr, h.d_mperm, h.n_multi, vals);
  else
    k4_multi<3><<<blocks, 256, 0, s>>>(h.d_side, h.d_mblk, h.d_mslot0, h.d_slot_tr, h.d_mperm, h.n_multi, vals);
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
