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

// the first two slots of a block (its range starts at an even slot: 16-B aligned in 3D, and
// always in 2D) as 16-B read-only loads
template <int D>
__device__ __forceinline__ void k4_load2(const double *__restrict__ side, int32_t s0, double (&l0)[D * D],
                                         double (&l1)[D * D]) {
  constexpr int DD = D * D;
  const double2 *p = reinterpret_cast<const double2 *>(side + (int64_t)s0 * DD);
  double t[2 * DD];
#pragma unroll
  for (int v = 0; v < DD; ++v) {
    const double2 x = __ldg(p + v);
    t[2 * v] = x.x;
    t[2 * v + 1] = x.y;
  }
#pragma unroll
  for (int e = 0; e < DD; ++e) {
    l0[e] = t[e];
    l1[e] = t[DD + e];
  }
}

// the slot sums of the two blocks of thread m (pass 1 and pass 2): a multi block has at least
// two slots, so the first two slots of both (and their orientation flags) are loaded in one
// round trip before any addition; further slots (tile edges and corners) follow in the fixed
// slot order (the sum is (L_0 + L_1) + L_2 + ..., as K4 always formed it)
template <int D>
__device__ __forceinline__ void k4_sum2(const double *__restrict__ side, const uint8_t *__restrict__ slot_tr,
                                        const K4Desc &d1, const K4Desc &d2, const double (&l)[4][D * D],
                                        double *acc1, double *acc2) {
  constexpr int DD = D * D;
  // l: the first two slots of both blocks, loaded by the caller
  // the two orientation flags of a block's first slots: one 2-B load (s0 even)
  const uint16_t f1 = __ldg(reinterpret_cast<const uint16_t *>(slot_tr + d1.s0));
  const uint16_t f2 = __ldg(reinterpret_cast<const uint16_t *>(slot_tr + d2.s0));
  const bool t0 = f1 & 0xff, t1 = f1 >> 8, t2 = f2 & 0xff, t3 = f2 >> 8;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      acc1[a * D + b] = (t0 ? l[0][b * D + a] : l[0][a * D + b]) + (t1 ? l[1][b * D + a] : l[1][a * D + b]);
      acc2[a * D + b] = (t2 ? l[2][b * D + a] : l[2][a * D + b]) + (t3 ? l[3][b * D + a] : l[3][a * D + b]);
    }
  const int ns1 = (d1.sn >> 17) & (K4_MAX_NS - 1), ns2 = (d2.sn >> 17) & (K4_MAX_NS - 1);
  for (int sl = d1.s0 + 2; sl < d1.s0 + ns1; ++sl) {
    const double *L = side + (int64_t)sl * DD;
    const bool tr = slot_tr[sl];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) acc1[a * D + b] += tr ? L[b * D + a] : L[a * D + b];
  }
  for (int sl = d2.s0 + 2; sl < d2.s0 + ns2; ++sl) {
    const double *L = side + (int64_t)sl * DD;
    const bool tr = slot_tr[sl];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) acc2[a * D + b] += tr ? L[b * D + a] : L[a * D + b];
  }
}

__device__ __forceinline__ K4Desc k4_ld_desc(const K4Desc *p) {
  const int4 v = __ldg(reinterpret_cast<const int4 *>(p));
  K4Desc d;
  d.off = (int64_t)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
  d.s0 = v.z;
  d.sn = (uint32_t)v.w;
  return d;
}

// Thread m: pass 1 writes K(I,J) of multi block m (blocks ordered by (I, J)); pass 2 writes
// K(J,I) of the m-th block in (J, I) order.  Both orders put neighbouring blocks of one CSR
// row in neighbouring lanes; the d-double row segments are stored warp-cooperatively from a
// shared-memory copy of the sums (whole sectors for runs of adjacent blocks).  Each pass's
// store target and slot range come from one 16-B descriptor (K4Desc, built on the host).
#ifndef IGA_K4_MINB
#define IGA_K4_MINB 3   // 3 CTAs of 256 per SM (85 registers): 0.547 ms at cfg5; 2 (110 registers) 0.585, 4 (64) 0.576
#endif
template <int D>
__global__ void __launch_bounds__(256, IGA_K4_MINB)
k4_multi(const double *__restrict__ side, const K4Desc *__restrict__ k4d, const uint8_t *__restrict__ slot_tr,
         int64_t n_multi, double *__restrict__ vals) {
  constexpr int DD = D * D;
  __shared__ double sacc[2][256 * DD];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + tid;
  const bool live = m < n_multi;
  K4Desc d1{-1, 0, 0}, d2{-1, 0, 0};
  double l[4][DD];
  if (live) {
    d1 = k4_ld_desc(k4d + m);
    d2 = k4_ld_desc(k4d + n_multi + m);
    k4_load2<D>(side, d1.s0, l[0], l[1]);
    k4_load2<D>(side, d2.s0, l[2], l[3]);
  }
  double acc1[DD], acc2[DD];
  if (live) k4_sum2<D>(side, slot_tr, d1, d2, l, acc1, acc2);
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
#ifdef IGA_EXPERIMENT_K4_ST_HINT   // CSR values are written once: L2 evict-first
          st_hint(vals + ob + (int64_t)idx * sstr + c, sacc[pass][(wbase + src) * DD + ra * D + cb], l2_policy_evict_first());
#else
          vals[ob + (int64_t)idx * sstr + c] = sacc[pass][(wbase + src) * DD + ra * D + cb];
#endif
        }
      }
    }
  };
  coop(live ? d1.off : -1, (int)(d1.sn & 0x1ffff), (d1.sn >> 31) != 0, 0);
  coop(live ? d2.off : -1, (int)(d2.sn & 0x1ffff), false, 1);
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
    k4_multi<2><<<blocks, 256, 0, s>>>(h.d_side, h.d_k4d, h.d_slot_tr, h.n_multi, vals);
  else
    k4_multi<3><<<blocks, 256, 0, s>>>(h.d_side, h.d_k4d, h.d_slot_tr, h.n_multi, vals);
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
