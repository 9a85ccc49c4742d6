// device_common.cuh — small device helpers shared by the libiga kernels.
#pragma once
#include <cuda_runtime.h>
#include "internal.h"

namespace iga {

// Nonzero B-spline basis values N[r] = N_{s-p+r,p}(u) and first derivatives on knot
// span s (Cox–de Boor triangle; derivative from the degree p-1 values:
// N'_{i,p} = p N_{i,p-1}/(U_{i+p}-U_i) - p N_{i+1,p-1}/(U_{i+p+1}-U_{i+1})).
__device__ __forceinline__ void bspline_eval(const double *U, int p, int s, double u, double *N, double *dN) {
  double left[IGA_MAXP + 1], right[IGA_MAXP + 1], Nd[IGA_MAXP + 1], Nm1[IGA_MAXP + 1];
  Nd[0] = 1.0;
  Nm1[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = u - U[s + 1 - j];
    right[j] = U[s + j] - u;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      double temp = Nd[r] / (right[r + 1] + left[j - r]);
      Nd[r] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    Nd[j] = saved;
    if (j == p - 1)
      for (int r = 0; r < p; ++r) Nm1[r] = Nd[r];
  }
  for (int r = 0; r <= p; ++r) {
    N[r] = Nd[r];
    int i = s - p + r;
    double t1 = (r >= 1) ? Nm1[r - 1] / (U[i + p] - U[i]) : 0.0;
    double t2 = (r <= p - 1) ? Nm1[r] / (U[i + p + 1] - U[i + 1]) : 0.0;
    dN[r] = p * (t1 - t2);
  }
}

// the same values with every loop fully unrolled up to IGA_MAXP and guarded by p, so the
// triangle lives in registers (no local-memory arrays); N, dN must hold IGA_MAXP+1 values
__device__ __forceinline__ void bspline_eval_reg(const double *U, int p, int s, double u, double *N, double *dN) {
  double left[IGA_MAXP + 1], right[IGA_MAXP + 1], Nd[IGA_MAXP + 1], Nm1[IGA_MAXP + 1];
#pragma unroll
  for (int r = 0; r <= IGA_MAXP; ++r) Nd[r] = Nm1[r] = left[r] = right[r] = 0.0;
  Nd[0] = 1.0;
  Nm1[0] = 1.0;
#pragma unroll
  for (int j = 1; j <= IGA_MAXP; ++j) {
    if (j <= p) {
      left[j] = u - U[s + 1 - j];
      right[j] = U[s + j] - u;
      double saved = 0.0;
#pragma unroll
      for (int r = 0; r < j; ++r) {
        double temp = Nd[r] / (right[r + 1] + left[j - r]);
        Nd[r] = saved + right[r + 1] * temp;
        saved = left[j - r] * temp;
      }
      Nd[j] = saved;
      if (j == p - 1) {
#pragma unroll
        for (int r = 0; r < j + 1; ++r) Nm1[r] = Nd[r];
      }
    }
  }
#pragma unroll
  for (int r = 0; r <= IGA_MAXP; ++r) {
    if (r <= p) {
      N[r] = Nd[r];
      const int i = s - p + r;
      const double t1 = (r >= 1) ? Nm1[r - 1] / (U[i + p] - U[i]) : 0.0;
      const double t2 = (r <= p - 1) ? Nm1[r] / (U[i + p + 1] - U[i + 1]) : 0.0;
      dN[r] = p * (t1 - t2);
    }
  }
}

template <int D>
__device__ __forceinline__ double det_inv(const double J[D][D], double G[D][D]) {
  if (D == 2) {
    double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    double id = 1.0 / det;
    G[0][0] = J[1][1] * id;
    G[0][1] = -J[0][1] * id;
    G[1][0] = -J[1][0] * id;
    G[1][1] = J[0][0] * id;
    return det;
  } else {
    double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    double id = 1.0 / det;
    G[0][0] = c00 * id;
    G[1][0] = c01 * id;
    G[2][0] = c02 * id;
    G[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
    G[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
    G[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
    G[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
    G[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
    G[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
    return det;
  }
}

__device__ __forceinline__ double bernstein1(int q, int k, double x) {
  double b = 1.0;
  for (int i = 1; i <= k; ++i) b = b * (q - k + i) / i;   // binom(q, k)
  double r = b;
  for (int i = 0; i < k; ++i) r *= x;
  for (int i = 0; i < q - k; ++i) r *= (1.0 - x);
  return r;
}

// ---- Eq. 38 (Ā_ij[a,b] = Ā_ji[b,a]) reduced contraction ("sym" layout) ----
// Part 1 pairs / outputs: the d(d+1)/2 index pairs (a,b), a <= b, diagonal first then
// (0,1), (0,2), (1,2); part 2: the d(d-1)/2 pairs a < b in the same order.
__host__ __device__ __forceinline__ constexpr int sym_index(int D, int a, int b) {   // a <= b
  return a == b ? a : (D == 2 ? 2 : (a == 0 ? 2 + b : 5));
}
__host__ __device__ __forceinline__ constexpr int anti_index(int D, int a, int b) {  // a < b
  return D == 2 ? 0 : (a == 0 ? b - 1 : 2);
}
__host__ __device__ __forceinline__ void sym_pair(int D, int o, int &a, int &b) {
  if (o < D) { a = b = o; return; }
  if (D == 2) { a = 0; b = 1; return; }
  a = o == 5 ? 1 : 0;
  b = o == 3 ? 1 : 2;
}
__host__ __device__ __forceinline__ void anti_pair(int D, int o, int &a, int &b) {
  if (D == 2) { a = 0; b = 1; return; }
  a = o == 2 ? 1 : 0;
  b = o == 0 ? 1 : 2;
}

// record the first degeneracy (flag[0] = code, flag[1] = tile/patch, flag[2] = node/point)
__device__ __forceinline__ void raise_flag(int *flag, int code, int a, int b) {
  if (atomicCAS(flag, 0, code) == 0) {
    flag[1] = a;
    flag[2] = b;
  }
}

// FP64 tensor core: D = A(8x4,row) * B(4x8,col) + C, per-lane fragments
// a = A[l/4][l%4], b = B[l%4][l/4], c = C[l/4][2(l%4)+{0,1}]  (verified, profiles/r01_fp64_ceiling.md)
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- bulk async copies (cp.async.bulk, SASS UBLKCP) + mbarrier pipelines ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// the same wait on a precomputed shared-window address (no address conversion in the loop)
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// bytes: multiple of 16; both addresses 16-B aligned.  Completion is signalled on `bar`.
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// thread-block cluster barrier halves and distributed shared memory
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
// generic address of the same shared-memory object in the cluster's CTA `rank`
template <typename T>
__device__ __forceinline__ T *cluster_map(T *p, int rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;\n" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<T *>(out);
}

// L2 cache policies (createpolicy) for bulk copies and stores
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void *smem, const void *gmem, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// (IGA_EXPERIMENT_ST_NOCLOBBER: no "memory" clobber, so the compiler may hoist the shared-memory
// loads of later stores above these global stores)
#ifndef IGA_EXPERIMENT_ST_NOCLOBBER
#define IGA_ST_CLOBBER : "memory"
#else
#define IGA_ST_CLOBBER
#endif
__device__ __forceinline__ void st_hint(double *p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) IGA_ST_CLOBBER);
}
__device__ __forceinline__ void st2_hint(double *p, double v0, double v1, uint64_t pol) {   // p 16-B aligned
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v0), "d"(v1), "l"(pol) : "memory");
}

// Fragment-major ("FM") operand layout of an R×K matrix for mma.m8n8k4:
// chunks of BR rows × 16 columns are contiguous (BR*16 doubles, ordered [row block][k
// chunk]); inside a chunk, 8-row group g and 4-column step kk hold the 32 values a warp
// loads as one fragment, in lane order lane = (row%8)*4 + k%4.  One bulk copy moves a
// chunk; one LDS.64 per lane (256 contiguous bytes per warp) loads a fragment.
__host__ __device__ __forceinline__ int64_t fm_index(int64_t r, int k, int BR, int nkc) {
  const int64_t rb = r / BR;
  const int rr = (int)(r - rb * BR);
  return ((rb * nkc + (k >> 4)) * BR + (rr & ~7)) * 16 + ((k >> 2) & 3) * 32 + ((rr & 7) << 2) + (k & 3);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace iga
