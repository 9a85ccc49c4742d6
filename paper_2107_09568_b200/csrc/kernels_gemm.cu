// kernels_gemm.cu — FP64 tensor-core contractions (SASS DMMA.8x8x4 via mma.sync;
// sm_100a has no FP64 tcgen05/wgmma kind — profiles/r01_fp64_ceiling.md).
//
// K3 (Eq. 58; "Step 3 is largely the most demanding step"):
//   local[M][N] = mat𝔎[M][K] · mat⟨Ā⟩[K][N],  M = Σ_p n_nz,p, K = d² n_π, N = d² n_tiles.
//   A = table (row-major, k_stride), B = coefficients stored N-major (coef[n][κ]).
// K5a (Eq. 73, "the product of the lookup table ... and the displacement DOF"):
//   W[n][κ] = Σ_row mat𝔎[row][κ] X[row][n], X generated on the fly from u, v and the
//   node map (never materialised).
//
// Tiling: CTA 128×64 output tile, 8 warps (4×2), warp tile 32×32 = 4×4 DMMA tiles,
// k-chunk 16 staged by cp.async in a 3-stage ring, smem rows padded to 20 doubles so
// the per-lane fragment loads (row l/4, col l%4) are bank-conflict free per half-warp.
// Epilogue staged through shared memory for coalesced 512-B row writes.
// Grid: M-blocks fastest, so the CTAs resident at one time share the B (coefficient)
// block and the table stays L2-resident (39.6 MB for cfg3/cfg5 < 126 MB L2).
#include "device_common.cuh"

namespace iga {

constexpr int BM = 128, BN = 64, BK = IGA_KCHUNK, SROW = BK + 4, STAGES = 3, NTHREADS = 256;
constexpr int WM = 32, WN = 32;                  // warp tile
constexpr int MI = WM / 8, NI = WN / 8;          // DMMA tiles per warp
constexpr int CROW = BN + 2;                     // epilogue staging row (doubles)
constexpr size_t GEMM_SMEM = sizeof(double) * (size_t)STAGES * (BM + BN) * SROW;
static_assert(GEMM_SMEM >= sizeof(double) * (size_t)BM * CROW, "epilogue staging must fit");

__device__ __forceinline__ void mma_chunk(const double *sA, const double *sB, int wm0, int wn0, int lane,
                                          int ksteps, double (&acc)[MI][NI][2]) {
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) {
    if (kk < ksteps) {
      double a[MI], b[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[mi] = sA[(wm0 + mi * 8 + fr) * SROW + kk * 4 + fc];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = sB[(wn0 + ni * 8 + fr) * SROW + kk * 4 + fc];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
}

__device__ __forceinline__ void load_tile_async(double *s, const double *g, int64_t row0, int64_t nrows,
                                                int rows, int64_t ld, int64_t col0, int tid) {
  // rows × BK doubles, 16-B chunks; out-of-range rows are clamped (results discarded)
  for (int i = tid; i < rows * (BK / 2); i += NTHREADS) {
    int r = i / (BK / 2), c2 = i % (BK / 2);
    int64_t gr = row0 + r;
    if (gr >= nrows) gr = nrows - 1;
    cp_async16(s + r * SROW + c2 * 2, g + gr * ld + col0 + c2 * 2);
  }
}

// C[M][ldc] = A[M][kstride] · B[N][kstride]ᵀ over ksteps*4 columns.
__global__ void __launch_bounds__(NTHREADS, 2)
k3_contract(const double *__restrict__ A, const double *__restrict__ B, double *__restrict__ C, int64_t M,
            int64_t N, int ksteps, int kstride, int64_t ldc) {
  extern __shared__ __align__(16) double smem[];
  double *sA = smem, *sB = smem + STAGES * BM * SROW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp >> 1) * WM, wn0 = (warp & 1) * WN;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int kcols = ksteps * 4;
  const int nchunks = (kcols + BK - 1) / BK;
  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) {
      load_tile_async(sA + s * BM * SROW, A, m0, M, BM, kstride, (int64_t)s * BK, tid);
      load_tile_async(sB + s * BN * SROW, B, n0, N, BN, kstride, (int64_t)s * BK, tid);
    }
    cp_async_commit();
  }
  for (int kc = 0; kc < nchunks; ++kc) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    int nxt = kc + STAGES - 1;
    if (nxt < nchunks) {
      int st = nxt % STAGES;
      load_tile_async(sA + st * BM * SROW, A, m0, M, BM, kstride, (int64_t)nxt * BK, tid);
      load_tile_async(sB + st * BN * SROW, B, n0, N, BN, kstride, (int64_t)nxt * BK, tid);
    }
    cp_async_commit();
    const int st = kc % STAGES;
    int steps = min(BK / 4, ksteps - kc * (BK / 4));
    mma_chunk(sA + st * BM * SROW, sB + st * BN * SROW, wm0, wn0, lane, steps, acc);
  }
  cp_async_wait<0>();
  __syncthreads();
  double *sC = smem;
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      int r = wm0 + mi * 8 + fr, c = wn0 + ni * 8 + 2 * fc;
      sC[r * CROW + c] = acc[mi][ni][0];
      sC[r * CROW + c + 1] = acc[mi][ni][1];
    }
  __syncthreads();
  for (int i = tid; i < BM * BN; i += NTHREADS) {
    int r = i / BN, c = i % BN;
    int64_t gr = m0 + r, gc = n0 + c;
    if (gr < M && gc < N) C[gr * ldc + gc] = sC[r * CROW + c];
  }
}

// K5a: W[n][κ] = Σ_r tableT[κ][r] X[r][n]; M' = kstride (κ), N' = n_tiles*d², K' = rows.
template <int D>
__global__ void __launch_bounds__(NTHREADS, 2)
k5a_wgemm(const double *__restrict__ AT, int64_t ldaT, int64_t Mrows, const int *__restrict__ node_map,
          int nl, const int *__restrict__ pairA, const int *__restrict__ pairB, const double *__restrict__ u,
          const double *__restrict__ v, int64_t N, double *__restrict__ W, int kstride) {
  extern __shared__ __align__(16) double smem[];
  double *sA = smem, *sB = smem + STAGES * BM * SROW;
  constexpr int DD = D * D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp >> 1) * WM, wn0 = (warp & 1) * WN;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t Mk = kstride;                    // rows of AT actually stored
  const int nchunks = (int)((Mrows + BK - 1) / BK);
  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  auto gen_X = [&](double *s, int64_t r0) {
    for (int i = tid; i < BN * BK; i += NTHREADS) {
      int c = i / BK, rr = i % BK;
      int64_t n = n0 + c, r = r0 + rr;
      double x = 0.0;
      if (n < N && r < Mrows) {
        int64_t t = n / DD;
        int ab = (int)(n % DD), a = ab / D, b = ab % D;
        int pa = pairA[r], pb = pairB[r];
        int64_t I = node_map[t * nl + pa], J = node_map[t * nl + pb];
        if (pa != pb) {
          x = u[I * D + a] * v[J * D + b] + u[J * D + b] * v[I * D + a];
        } else if (a < b) {
          x = u[I * D + a] * v[I * D + b] + u[I * D + b] * v[I * D + a];
        } else if (a == b) {
          x = u[I * D + a] * v[I * D + a];
        }
      }
      s[c * SROW + rr] = x;
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) {
      load_tile_async(sA + s * BM * SROW, AT, m0, Mk, BM, ldaT, (int64_t)s * BK, tid);
      gen_X(sB + s * BN * SROW, (int64_t)s * BK);
    }
    cp_async_commit();
  }
  for (int kc = 0; kc < nchunks; ++kc) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    int nxt = kc + STAGES - 1;
    if (nxt < nchunks) load_tile_async(sA + (nxt % STAGES) * BM * SROW, AT, m0, Mk, BM, ldaT, (int64_t)nxt * BK, tid);
    cp_async_commit();
    const int st = kc % STAGES;
    mma_chunk(sA + st * BM * SROW, sB + st * BN * SROW, wm0, wn0, lane, BK / 4, acc);
    if (nxt < nchunks) gen_X(sB + (nxt % STAGES) * BN * SROW, (int64_t)nxt * BK);
  }
  cp_async_wait<0>();
  __syncthreads();
  double *sC = smem;
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      int r = wm0 + mi * 8 + fr, c = wn0 + ni * 8 + 2 * fc;
      sC[r * CROW + c] = acc[mi][ni][0];
      sC[r * CROW + c + 1] = acc[mi][ni][1];
    }
  __syncthreads();
  for (int i = tid; i < BM * BN; i += NTHREADS) {   // transposed write W[n][κ], κ contiguous
    int c = i / BM, r = i % BM;
    int64_t gk = m0 + r, gn = n0 + c;
    if (gk < Mk && gn < N) W[gn * kstride + gk] = sC[r * CROW + c];
  }
}

cudaError_t launch_contraction(const Handle &h, const double *A, const double *B, double *C, int64_t M,
                               int64_t N, int K, int kstride, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_contract, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    attr = true;
  }
  int ksteps = (K + 3) / 4;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  k3_contract<<<grid, NTHREADS, GEMM_SMEM, s>>>(A, B, C, M, N, ksteps, kstride, N);
  return cudaGetLastError();
}

cudaError_t launch_sens_W(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s) {
  int64_t N = h.n_tiles * h.d * h.d;
  int64_t ldaT = (h.M + BK - 1) / BK * BK;
  dim3 grid((unsigned)((h.kstride + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  if (h.d == 2) {
    cudaFuncSetAttribute(k5a_wgemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    k5a_wgemm<2><<<grid, NTHREADS, GEMM_SMEM, s>>>(h.d_tableT, ldaT, h.M, h.d_node_map, h.n_local_ctrl, h.d_pairA,
                                                   h.d_pairB, u, v, N, W, h.kstride);
  } else {
    cudaFuncSetAttribute(k5a_wgemm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    k5a_wgemm<3><<<grid, NTHREADS, GEMM_SMEM, s>>>(h.d_tableT, ldaT, h.M, h.d_node_map, h.n_local_ctrl, h.d_pairA,
                                                   h.d_pairB, u, v, N, W, h.kstride);
  }
  return cudaGetLastError();
}

}  // namespace iga
