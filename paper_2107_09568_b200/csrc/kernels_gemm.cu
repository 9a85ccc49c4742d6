// kernels_gemm.cu — FP64 tensor-core contractions (SASS DMMA.8x8x4 via mma.sync;
// sm_100a has no FP64 tcgen05/wgmma kind — profiles/r01_fp64_ceiling.md).
//
// K3 (Eq. 58; "Step 3 is largely the most demanding step"):
//   nzdata[M][N] = mat𝔎[M][K] · mat⟨Ā⟩[K][N],  M = Σ_p n_nz,p, K = d² n_π, N = d² n_tiles,
//   evaluated in the Eq. 38-reduced form of DESIGN.md §6 (symmetric part: [𝔎_ii | 𝔎_ij + 𝔎_ji]
//   against the symmetric coefficient halves; antisymmetric part: 𝔎_ij − 𝔎_ji against the
//   antisymmetric halves; 45/81 of the multiply-adds in 3D), with the scatter of step 4
//   (reading R9) fused into the epilogue: each (row, tile) d×d block goes
//   straight to its two CSR positions (I,J) and (J,I) when it is the block's only
//   contribution, else to a side slot that K4 sums.  The 12 GB nzdata intermediate of cfg5
//   is never written.
// K5x / K5a (Eq. 73, "the product of the lookup table ... and the displacement DOF"):
//   X̃ (the coefficient of every local entry in uᵀK^πv, symmetric / antisymmetric combinations)
//   is written by the memory-bound K5x; K5a contracts it with the reduced table:
//   Y[n][κ] = Σ_row tab[row][κ] X̃[row][n].
//
// Operands live in HBM in the fragment-major layout of device_common.cuh (fm_index):
// every k-chunk of a CTA tile is one contiguous block moved by ONE cp.async.bulk
// (UBLKCP) into a ring of shared-memory stages guarded by mbarriers, and every DMMA
// fragment is one conflict-free 256-B LDS.64 per warp.
//
// DMMA issue: ptxas gives every DMMA a fixed 15-cycle stall plus a NOP, so one warp
// issues at most one DMMA per 16 cycles; an SM needs ~16 MMA warps to keep its FP64 tensor
// pipe busy.  K3: 64×72 CTA tiles, 4 MMA warps, 4 CTAs per SM, the same warps run the
// scatter after the main loop (co-resident CTAs keep the pipe busy meanwhile).  K5a: one
// CTA per 72-column N-block over all κ rows, 16 MMA warps.  Both: the last warp to release
// a stage refills it.
#include "device_common.cuh"

namespace iga {

constexpr int BK = IGA_KCHUNK;     // 16
constexpr int BN = IGA_GEMM_BN;    // 72
constexpr int NI = BN / 8;         // 9 DMMA column tiles per warp
constexpr int MI = 2;              // 2 DMMA row tiles per warp (16 rows)
constexpr int N_MMA_WARPS = IGA_K5_BM / 16;                                // K5a: 16
constexpr int BM = 16 * N_MMA_WARPS;                                        // 256 (K5a κ rows)
constexpr int K3_BM = IGA_K3_BM, K3_WARPS = K3_BM / 16;                     // K3: 64 rows, 4 MMA warps
constexpr int K3_CL = IGA_K3_CL;
#ifdef IGA_K3_TILE_UNROLL
constexpr int K3_TILE_UNROLL = IGA_K3_TILE_UNROLL;
#endif                                            // K3 CTAs per cluster (EPI 3)
static_assert(K3_CL == 1 || (K3_CL * K3_BM <= 65536 && K3_CL <= 8 && K3_BM == 64), "cluster row blocks: cperm is uint16, pk packs the rank in 3 bits above the row");
static_assert(K3_BM == 64 || K3_BM == 128, "K3 row blocks: 64 (product) or 128 rows; other shapes are not supported by every epilogue");
static_assert(BM == IGA_K5_BM, "K5a CTA rows");
constexpr int K5_X_CHUNK_ = BN * BK;                                        // doubles per X chunk

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// Fragment loads: sA/sB are FM chunks, g0 = first 8-row group of the warp in sA; the k-step
// loops are template-unrolled so that the fragment loads of step kk+1 are scheduled under the
// DMMAs of step kk.
// Eq. 38-reduced contraction: the GEMM columns are part 1 (P1 pairs × n_π,
// against the symmetric outputs = DMMA column tiles [0, 6)) then part 2 (P2 pairs × n_π,
// against the antisymmetric outputs = column tiles [6, NE), NE = 9 in 3D, 8 in 2D).
// KS k-steps from step kk0 of a chunk, row groups [MI0, MI0 + MIC), column tiles [LO, HI).
template <int KS, int MI0, int MIC, int LO, int HI>
__device__ __forceinline__ void mma_steps(const double *__restrict__ sA, const double *__restrict__ sB, int g0,
                                          int lane, int kk0, double (&acc)[MI][NI][2]) {
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int k = kk0 + kk;
    double a[MI], b[NI];
#pragma unroll
    for (int mi = MI0; mi < MI0 + MIC; ++mi) a[mi] = sA[((g0 + mi) * 4 + k) * 32 + lane];
#pragma unroll
    for (int ni = LO; ni < HI; ++ni) b[ni] = sB[(ni * 4 + k) * 32 + lane];
#pragma unroll
    for (int mi = MI0; mi < MI0 + MIC; ++mi)
#pragma unroll
      for (int ni = LO; ni < HI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

template <int MI0, int MIC, int LO, int HI>
__device__ __forceinline__ void mma_steps_n(const double *__restrict__ sA, const double *__restrict__ sB, int g0,
                                            int lane, int kk0, int n, double (&acc)[MI][NI][2]) {
  switch (n) {
    case 1: mma_steps<1, MI0, MIC, LO, HI>(sA, sB, g0, lane, kk0, acc); break;
    case 2: mma_steps<2, MI0, MIC, LO, HI>(sA, sB, g0, lane, kk0, acc); break;
    case 3: mma_steps<3, MI0, MIC, LO, HI>(sA, sB, g0, lane, kk0, acc); break;
    case 4: mma_steps<4, MI0, MIC, LO, HI>(sA, sB, g0, lane, kk0, acc); break;
    default: break;
  }
}

// one K3 chunk: ns k-steps of which [0, j) belong to part 1 and [j, ns) to part 2
template <int MIC, int NE>
__device__ __forceinline__ void k3_chunk(const double *__restrict__ sA, const double *__restrict__ sB, int g0, int lane,
                                         int ns, int j, double (&acc)[MI][NI][2]) {
  if (j >= 4 && ns == 4) {
    mma_steps<4, 0, MIC, 0, 6>(sA, sB, g0, lane, 0, acc);
  } else if (j == 0 && ns == 4) {
    mma_steps<4, 0, MIC, 6, NE>(sA, sB, g0, lane, 0, acc);
  } else {
    mma_steps_n<0, MIC, 0, 6>(sA, sB, g0, lane, 0, j < ns ? j : ns, acc);
    if (j < ns) mma_steps_n<0, MIC, 6, NE>(sA, sB, g0, lane, j, ns - j, acc);
  }
}

// ---- K3 main loop, software-pipelined across chunk boundaries ----------------------------
// The stage hand-over (release atomic, the wait for the next stage, the first fragment loads
// of the next chunk) used to sit between the last DMMA of one chunk and the first of the
// next: ~13% of the MMA warps' time with no DMMA of theirs in the pipe (ncu source view,
// profiles/r02_k3_pipeline.md).  Here the last k-step's fragments are loaded and consumed
// into registers first, the stage is released, the next stage awaited and its k-step-0
// fragments loaded, and only then the last k-step's DMMAs are issued, so the hand-over runs
// under 12 (part 1) or 6 (part 2) DMMAs.
template <int MIC, int LO, int HI>
__device__ __forceinline__ void frag_load(const double *__restrict__ sA, const double *__restrict__ sB, int g0, int lane,
                                          int k, double (&a)[MI], double (&b)[NI]) {
#pragma unroll
  for (int mi = 0; mi < MIC; ++mi) a[mi] = sA[((g0 + mi) * 4 + k) * 32 + lane];
#pragma unroll
  for (int ni = LO; ni < HI; ++ni) b[ni] = sB[(ni * 4 + k) * 32 + lane];
}
template <int MIC, int LO, int HI>
__device__ __forceinline__ void frag_mma(const double (&a)[MI], const double (&b)[NI], double (&acc)[MI][NI][2]) {
#ifdef IGA_EXPERIMENT_K3_NI_MAJOR
#pragma unroll
  for (int ni = LO; ni < HI; ++ni)
#pragma unroll
    for (int mi = 0; mi < MIC; ++mi) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
#else
#pragma unroll
  for (int mi = 0; mi < MIC; ++mi)
#pragma unroll
    for (int ni = LO; ni < HI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
#endif
}
// a real instruction reads every fragment register, so the warp passes this point only after
// all its shared-memory loads of the stage have returned (the stage may then be released)
template <int MIC, int LO, int HI>
__device__ __forceinline__ void frag_touch(const double (&a)[MI], const double (&b)[NI]) {
  uint32_t z = 0;
#pragma unroll
  for (int mi = 0; mi < MIC; ++mi) z |= (uint32_t)__double2loint(a[mi]);
#pragma unroll
  for (int ni = LO; ni < HI; ++ni) z |= (uint32_t)__double2loint(b[ni]);
  asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %0, 0x7ff8dead;\n @p nanosleep.u32 1;\n}\n" ::"r"(z) : "memory");
}
// lane 0 takes a ticket on the stage's release counter (monotonic: the KW-th ticket of each
// round belongs to the last warp to release the stage, which refills it)
__device__ __forceinline__ uint32_t k3_release(uint32_t counter, int lane) {
  uint32_t t = 0;
  asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %2, 0;\n @p atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;\n}\n"
               : "+r"(t)
               : "r"(counter), "r"(lane)
               : "memory");
  return t;
}
// k-step-0 fragments of a chunk whose first step lies in part 1 (p1) or part 2
template <int NE>
__device__ __forceinline__ void frag_load_first(const double *__restrict__ sA, const double *__restrict__ sB, int g0,
                                                int lane, bool p1, double (&a)[MI], double (&b)[NI]) {
  if (p1) frag_load<MI, 0, 6>(sA, sB, g0, lane, 0, a, b);
  else frag_load<MI, 6, NE>(sA, sB, g0, lane, 0, a, b);
}
// a full chunk (4 k-steps of one part, both row groups live); ca/cb hold its k-step 0 on
// entry and the next chunk's k-step 0 on exit.  Returns lane 0's release ticket.
template <int LO, int HI, int NE, int KW, class Refill>
__device__ __forceinline__ void k3_fast_chunk(const double *__restrict__ sA, const double *__restrict__ sB,
                                              const double *__restrict__ sAn, const double *__restrict__ sBn, int g0,
                                              int lane, double (&ca)[MI], double (&cb)[NI], double (&acc)[MI][NI][2],
                                              uint32_t counter, uint32_t full_next, uint32_t ph_next, bool more,
                                              bool p1n, Refill &&refill) {
  double a1[MI], b1[NI];
  frag_load<MI, LO, HI>(sA, sB, g0, lane, 1, a1, b1);
  frag_mma<MI, LO, HI>(ca, cb, acc);
  frag_load<MI, LO, HI>(sA, sB, g0, lane, 2, ca, cb);
  frag_mma<MI, LO, HI>(a1, b1, acc);
  frag_load<MI, LO, HI>(sA, sB, g0, lane, 3, a1, b1);
  frag_mma<MI, LO, HI>(ca, cb, acc);
#ifndef IGA_EXPERIMENT_K3_NOTOUCH
  frag_touch<MI, LO, HI>(a1, b1);
#endif
  const uint32_t ticket = k3_release(counter, lane);
#ifdef IGA_EXPERIMENT_K3_LATEWAIT
  if (lane == 0 && ticket % KW == KW - 1) refill();
  frag_mma<MI, LO, HI>(a1, b1, acc);
  if (more) {
    mbar_wait_a(full_next, ph_next);
    frag_load_first<NE>(sAn, sBn, g0, lane, p1n, ca, cb);
  }
#else
  if (more) {
    mbar_wait_a(full_next, ph_next);
    frag_load_first<NE>(sAn, sBn, g0, lane, p1n, ca, cb);
  }
  if (lane == 0 && ticket % KW == KW - 1) refill();   // the last warp to release a stage refills it
  frag_mma<MI, LO, HI>(a1, b1, acc);
#endif
}

// one d-double row segment of a CSR block row: the 16-B aligned pair goes out as one
// 128-bit store (2 store instructions per 3D row instead of 3)
template <int D>
__device__ __forceinline__ void store_row(double *p, double x0, double x1, double x2) {
  if (D == 3) {
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      *reinterpret_cast<double2 *>(p) = make_double2(x0, x1);
      p[2] = x2;
    } else {
      p[0] = x0;
      *reinterpret_cast<double2 *>(p + 1) = make_double2(x1, x2);
    }
  } else {
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      *reinterpret_cast<double2 *>(p) = make_double2(x0, x1);
    } else {
      p[0] = x0;
      p[1] = x1;
    }
  }
}

// one d-double CSR row segment with the L2 evict-first policy (CSR values are written once)
template <int D>
__device__ __forceinline__ void store_seg_hint(double *p, const double (&x)[D], uint64_t pol) {
  const bool al = (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  if (D == 3) {
    if (al) {
      st2_hint(p, x[0], x[1], pol);
      st_hint(p + 2, x[D - 1], pol);
    } else {
      st_hint(p, x[0], pol);
      st2_hint(p + 1, x[1], x[D - 1], pol);
    }
  } else {
    if (al) {
      st2_hint(p, x[0], x[1], pol);
    } else {
      st_hint(p, x[0], pol);
      st_hint(p + 1, x[1], pol);
    }
  }
}

// Register-direct fused scatter (R9) of one K3 MMA warp.  The accumulator
// fragment of lane (fr, fc) = (lane / 4, lane % 4) holds, for rows fr and fr + 8 of the
// warp's 16 rows and tiles tl = hh·8 + 2fc + e, ALL sym / anti outputs of each (row, tile)
// block (the sym column tiles of DESIGN §6 are per output component, their columns per
// tile), so L_t[a][b] = L⁺ ± L⁻ is formed in registers and stored straight to its two CSR
// positions: K(I,J) = L (diagonal rows: the upper triangle mirrored) and K(J,I) = Lᵀ, or to
// the block's side slot when several contributions share it (emap < 0, summed by K4).  No
// shared-memory staging, no CTA barrier and no shuffles: a warp scatters as soon as its own
// main loop ends, while the other warps of its SM sub-partition keep the DMMA pipe busy.
template <int D>
__device__ __forceinline__ void k3_direct_scatter(const double (&acc)[MI][NI][2], int warp, int lane, int64_t m0,
                                                  int64_t t0, int64_t M, int64_t n_tiles, double *__restrict__ out,
                                                  const int32_t *__restrict__ pairA, const int32_t *__restrict__ pairB,
                                                  const int32_t *__restrict__ emap,
                                                  const int64_t *__restrict__ rowinfo, int nl,
                                                  double *__restrict__ side) {
  constexpr int DD = D * D, NP1 = D * (D + 1) / 2, NH = D == 3 ? 1 : 2, NT = 2 * NH;   // NT tiles per lane
  const int fr = lane >> 2, fc = lane & 3;
  const uint64_t pol = l2_policy_evict_first();
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    // this row's map loads first (one dependent level: pair → rowinfo)
    const int64_t r = m0 + warp * 8 * MI + mi * 8 + fr;
    if (r >= M) break;   // rows of the warp ascend: the rest is padding
    const int A = pairA[r], B = pairB[r];
    int32_t ev[NT];
    int64_t riA[NT], riB[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int tl = (k >> 1) * 8 + 2 * fc + (k & 1);
      const int64_t t = t0 + tl < n_tiles ? t0 + tl : n_tiles - 1;
      ev[k] = emap[t * M + r];
      riA[k] = rowinfo[t * nl + A];
      riB[k] = rowinfo[t * nl + B];
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int hh = k >> 1, e = k & 1, tl = hh * 8 + 2 * fc + e;
      if (t0 + tl >= n_tiles) continue;
      double L[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          const int lo = a < b ? a : b, hi = a < b ? b : a;
          const double sp = acc[mi][sym_index(D, lo, hi) * NH + hh][e];
          if (a == b) {
            L[a][b] = sp;
          } else {
            const double am = acc[mi][(NP1 + anti_index(D, lo, hi)) * NH + hh][e];
            L[a][b] = a < b ? sp + am : sp - am;
          }
        }
      const int32_t v = ev[k];
      if (v < 0) {   // one of several contributions: side slot, summed by K4
        double *o = side + (int64_t)(-v - 1) * DD;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) o[a * D + b] = L[a][b];
        continue;
      }
      const bool diag = A == B;
      if (riA[k] >= 0) {   // K(I,J) = L (riA < 0: row of another shard)
        double *p = out + DD * (riA[k] >> 24) + D * (v & 0xffff);
        const int64_t str = D * (riA[k] & 0xffffff);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double x[D];
#pragma unroll
          for (int b = 0; b < D; ++b) x[b] = diag && a > b ? L[b][a] : L[a][b];
          store_seg_hint<D>(p + a * str, x, pol);
        }
      }
      if (!diag && riB[k] >= 0) {   // K(J,I) = Lᵀ
        double *p = out + DD * (riB[k] >> 24) + D * (v >> 16);
        const int64_t str = D * (riB[k] & 0xffffff);
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double x[D];
#pragma unroll
          for (int a = 0; a < D; ++a) x[a] = L[a][b];
          store_seg_hint<D>(p + b * str, x, pol);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// K3: one CTA per 64×72 output tile, 4 MMA warps of 16×72, 3-stage bulk-copy ring
// refilled by the last warp to release a stage, 4 CTAs per SM (16 MMA warps: the DMMA
// pipe stays fed while co-resident CTAs run their epilogues; measured 128-row/2-CTA
// 22.1 ms, 96-row/3-CTA 21.8 ms, 64-row/4-CTA 21.3 ms at cfg5).  After the main loop the
// same warps stage the tile in shared memory and scatter it.
#ifndef IGA_K3_STAGES
#define IGA_K3_STAGES 3
#endif
constexpr int K3_STAGES = IGA_K3_STAGES;
constexpr int K3_A_CHUNK = K3_BM * BK, K3_B_CHUNK = BN * BK;          // doubles
constexpr int K3_CROW = BN + 1;                                        // epilogue pitch (odd)
constexpr size_t K3_STAGE_BYTES = sizeof(double) * (size_t)K3_STAGES * (K3_A_CHUNK + K3_B_CHUNK);
// epilogue staging: the tile (odd pitch) and, for the apply epilogue (EPI 2), its run sums (2 tiles)
template <int EPI>
constexpr size_t k3_epi_bytes() { return sizeof(double) * (size_t)K3_BM * (K3_CROW + (EPI == 2 ? 8 * 3 : 0)); }
template <int EPI>
constexpr size_t k3_off_bar() { return K3_STAGE_BYTES > k3_epi_bytes<EPI>() ? K3_STAGE_BYTES : k3_epi_bytes<EPI>(); }
#ifndef IGA_K3_SMEM_EXTRA
#define IGA_K3_SMEM_EXTRA 0   // experiment knob: unused bytes that cap the CTAs per SM
#endif
template <int EPI>
constexpr size_t k3_smem() { return k3_off_bar<EPI>() + K3_STAGES * (sizeof(uint64_t) + sizeof(int)) + IGA_K3_SMEM_EXTRA; }
#ifndef IGA_K3_MI
#define IGA_K3_MI 2   // 8-row DMMA groups per K3 MMA warp for EPI 0/1 (the apply epilogue keeps 2)
#endif
// per-epilogue K3 shape: MMA warps of 8·MI rows, threads = 32·warps, CTAs per SM hint
template <int EPI>
struct K3Cfg {
  static constexpr int KMI = EPI == 2 ? 2 : IGA_K3_MI;
  static constexpr int WARPS = K3_BM / (8 * KMI), THREADS = 32 * WARPS;
#ifdef IGA_K3_MINB   // experiment knob: CTAs per SM (register cap)
  static constexpr int MINB = IGA_K3_MINB;
#else
  static constexpr int MINB = KMI == 2 ? 256 / K3_BM : 3;
#endif
  static_assert(THREADS % K3_BM == 0, "epilogue: whole threads per row");
};

__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); }

// matrix-free apply (EPI = 2, NEXT N1): u, the partial buffer and the run maps
struct ApplyArgs {
  const double *u;
  double *part;
  int64_t P;
  const uint16_t *g1len, *g2len;
  const int32_t *g1slot, *g2slot, *node_map;
};

// EPI = 0: local[M][N] (nzdata, Eq. 58) ; EPI = 1: fused CSR scatter (+ side slots);
// EPI = 2: matrix-free apply y = K^π u (Eq. 74): block products summed into partial slots
template <int D, int EPI>
__global__ void __launch_bounds__(K3Cfg<EPI>::THREADS, K3Cfg<EPI>::MINB)
k3_contract(const double *__restrict__ tabA, const double *__restrict__ coef, int nkc, int ksteps, int ksplit, int64_t M,
            int64_t n_tiles, double *__restrict__ out, const int32_t *__restrict__ pairA,
            const int32_t *__restrict__ pairB, const int32_t *__restrict__ emap, const int64_t *__restrict__ rowinfo,
            int nl, double *__restrict__ side, const uint8_t *__restrict__ tperm, const uint16_t *__restrict__ cperm,
            const int4 *__restrict__ rowdesc, const ApplyArgs ap) {
  // tiles per CTA (sym layout: 8 in 3D, 16 in 2D), per epilogue thread; part-2 column tiles end
  constexpr int KMI = K3Cfg<EPI>::KMI, KW = K3Cfg<EPI>::WARPS, KT = K3Cfg<EPI>::THREADS;
  constexpr int DD = D * D, TPC = D == 3 ? 8 : 16, TPT = TPC / (KT / K3_BM), NE = D == 3 ? 9 : 8;
  extern __shared__ __align__(128) double smem[];
  double *sA = smem, *sB = smem + K3_STAGES * K3_A_CHUNK;
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + k3_off_bar<EPI>());
  int *released = reinterpret_cast<int *>(full + K3_STAGES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mb = blockIdx.x, nb = blockIdx.y, m0 = mb * K3_BM, t0 = nb * TPC;
  const double *gA = tabA + mb * nkc * K3_A_CHUNK, *gB = coef + nb * nkc * K3_B_CHUNK;
  // epilogue ownership: row er of the tile, tiles [et0, et0 + TPT) of the CTA
  const int er = tid % K3_BM, et0 = (tid / K3_BM) * TPT;
  const int64_t r = m0 + er;
  if (tid == 0) {
    for (int s = 0; s < K3_STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    mbar_fence_init();
  }
#ifndef IGA_EXPERIMENT_NO_PREFETCH
  if ((EPI == 1 || EPI == 3) && r < M)   // warm L2 with the epilogue's maps while the main loop runs
    for (int tl = et0; tl < et0 + TPT && t0 + tl < n_tiles; ++tl) prefetch_l2(emap + (t0 + tl) * M + r);
#endif
  __syncthreads();
  auto produce = [&](int kc) {
    const int st = kc % K3_STAGES;
#ifdef IGA_EXPERIMENT_K3_PART_B
    // experiment (profiles/r02_k3_pipeline.md, not faster): copy only the column tiles this
    // chunk's k-steps multiply (part 1: tiles [0, 6), part 2: [6, NE); the rest of the block
    // is zero and never read), a quarter less L2 -> SM traffic
    const int ps0 = kc * (BK / 4), pns = min(BK / 4, ksteps - ps0), pj = max(0, min(ksplit - ps0, pns));
    const int b_off = pj == 0 ? 6 * 4 * 32 : 0, b_len = (pj >= pns ? 6 : pj == 0 ? NE - 6 : NE) * 4 * 32;
#else
    const int b_off = 0, b_len = K3_B_CHUNK;
#endif
    mbar_expect_tx(&full[st], (K3_A_CHUNK + b_len) * 8);
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS   // keep the re-read table in L2 against the CSR store stream
    bulk_g2s_hint(sA + st * K3_A_CHUNK, gA + (int64_t)kc * K3_A_CHUNK, K3_A_CHUNK * 8, &full[st], l2_policy_evict_last());
#else
    bulk_g2s(sA + st * K3_A_CHUNK, gA + (int64_t)kc * K3_A_CHUNK, K3_A_CHUNK * 8, &full[st]);
#endif
    bulk_g2s(sB + st * K3_B_CHUNK + b_off, gB + (int64_t)kc * K3_B_CHUNK + b_off, b_len * 8, &full[st]);
  };
  if (tid == 0)
    for (int s = 0; s < K3_STAGES && s < nkc; ++s) produce(s);
  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  // 8-row groups of this warp that hold table rows < M (the rest is the zero padding of
  // the last row block: no DMMA is issued for it)
  const int64_t wr0 = m0 + warp * 8 * KMI;
  const int nmi = wr0 >= M ? 0 : (KMI == 2 && wr0 + 8 < M ? 2 : 1);
#ifdef IGA_EXPERIMENT_K3_PIPE   // measured slower (profiles/r02_k3_pipeline.md); the plain chunk loop below is the product
  if constexpr (KMI == 2) {
    const uint32_t full_a = smem_u32(full), rel_a = smem_u32(released);
    const int g0 = warp * KMI;
    if (nmi == 2) {
      // both row groups live (every warp but the last row block's tail): software-pipelined
      // across chunk boundaries (see k3_fast_chunk)
      double ca[MI], cb[NI];
      mbar_wait_a(full_a, 0);
      frag_load_first<NE>(sA, sB, g0, lane, 0 < ksplit, ca, cb);
      int st = 0;
      uint32_t ph = 0;
      for (int kc = 0; kc < nkc; ++kc) {
        const double *a_st = sA + st * K3_A_CHUNK, *b_st = sB + st * K3_B_CHUNK;
        const int stn = st + 1 == K3_STAGES ? 0 : st + 1;
        const uint32_t phn = stn == 0 ? ph ^ 1u : ph;
        const double *a_nx = sA + stn * K3_A_CHUNK, *b_nx = sB + stn * K3_B_CHUNK;
        const int s0 = kc * (BK / 4), ns = min(BK / 4, ksteps - s0), j = max(0, min(ksplit - s0, ns));
        const bool more = kc + 1 < nkc, p1n = s0 + BK / 4 < ksplit;
        auto refill = [&]() {
          if (kc + K3_STAGES < nkc) produce(kc + K3_STAGES);
        };
        if (ns == 4 && j == 4) {
          k3_fast_chunk<0, 6, NE, KW>(a_st, b_st, a_nx, b_nx, g0, lane, ca, cb, acc, rel_a + 4 * st, full_a + 8 * stn, phn,
                                      more, p1n, refill);
        } else if (ns == 4 && j == 0) {
          k3_fast_chunk<6, NE, NE, KW>(a_st, b_st, a_nx, b_nx, g0, lane, ca, cb, acc, rel_a + 4 * st, full_a + 8 * stn,
                                       phn, more, p1n, refill);
        } else {
          // mixed or short chunk: k-step 0 from the carried fragments, the rest as before;
          // the hand-over follows the last DMMA
          const int j1 = max(j, 1);
          if (j > 0) frag_mma<2, 0, 6>(ca, cb, acc);
          else frag_mma<2, 6, NE>(ca, cb, acc);
          mma_steps_n<0, 2, 0, 6>(a_st, b_st, g0, lane, 1, j1 - 1, acc);
          mma_steps_n<0, 2, 6, NE>(a_st, b_st, g0, lane, j1, ns - j1, acc);
          const uint32_t ticket = k3_release(rel_a + 4 * st, lane);
          if (lane == 0 && ticket % KW == KW - 1) refill();
          if (more) {
            mbar_wait_a(full_a + 8 * stn, phn);
            frag_load_first<NE>(a_nx, b_nx, g0, lane, p1n, ca, cb);
          }
        }
        st = stn;
        ph = phn;
      }
    } else {
      // the last row block's warps with one or no live row group: plain chunk loop, same
      // release protocol
      for (int kc = 0; kc < nkc; ++kc) {
        const int st = kc % K3_STAGES;
        mbar_wait_a(full_a + 8 * st, (kc / K3_STAGES) & 1);
        const int s0 = kc * (BK / 4), ns = min(BK / 4, ksteps - s0), j = max(0, min(ksplit - s0, ns));
        if (nmi == 1) k3_chunk<1, NE>(sA + st * K3_A_CHUNK, sB + st * K3_B_CHUNK, g0, lane, ns, j, acc);
        const uint32_t ticket = k3_release(rel_a + 4 * st, lane);
        if (lane == 0 && ticket % KW == KW - 1 && kc + K3_STAGES < nkc) produce(kc + K3_STAGES);
      }
    }
  } else
#endif
  {
  for (int kc = 0; kc < nkc; ++kc) {
    const int st = kc % K3_STAGES;
    mbar_wait(&full[st], (kc / K3_STAGES) & 1);
    const double *a_st = sA + st * K3_A_CHUNK, *b_st = sB + st * K3_B_CHUNK;
    // k-steps of this chunk and the first one of part 2 (Eq. 38-reduced contraction)
#ifdef IGA_EXPERIMENT_K3_INTERLEAVE   // timing only (wrong K): part-2 chunks interleaved 1:2 with part-1 chunks
    const int s0 = kc * (BK / 4), ns = min(BK / 4, ksteps - s0), j = kc % 3 == 2 ? 0 : ns;
#else
    const int s0 = kc * (BK / 4), ns = min(BK / 4, ksteps - s0), j = max(0, min(ksplit - s0, ns));
#endif
    if (nmi == 2) k3_chunk<2, NE>(a_st, b_st, warp * KMI, lane, ns, j, acc);
    else if (nmi == 1) k3_chunk<1, NE>(a_st, b_st, warp * KMI, lane, ns, j, acc);
#ifdef IGA_EXPERIMENT_K3_CHEAPREL
    {
      const uint32_t ticket = k3_release(smem_u32(released) + 4 * st, lane);
      if (lane == 0 && ticket % KW == KW - 1 && kc + K3_STAGES < nkc) produce(kc + K3_STAGES);
    }
#else
    __syncwarp();
    if (lane == 0) {   // the last warp to release a stage refills it
      __threadfence_block();
      if (atomicAdd(&released[st], 1) == KW - 1) {
        released[st] = 0;
        __threadfence_block();
        if (kc + K3_STAGES < nkc) produce(kc + K3_STAGES);
      }
    }
#endif
  }
  }
#ifdef IGA_EXPERIMENT_K3_DIRECT
  if constexpr (EPI == 1 && KMI == 2) {   // every thread returns here: no barrier below is reached
    k3_direct_scatter<D>(acc, warp, lane, m0, t0, M, n_tiles, out, pairA, pairB, emap, rowinfo, nl, side);
    return;
  }
#endif
  __syncthreads();   // all stages consumed: stage the tile in shared memory
  double *sC = smem;
  {
    const int fr = lane >> 2, fc = lane & 3;
#ifdef IGA_EXPERIMENT_K3_BARE
    double sum = 0.0;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) sum += acc[mi][ni][0] + acc[mi][ni][1];
    if (sum == 1.2345) out[0] = sum;
    return;
#endif
    // stage the tile-major L_t[a][b] (column tl·DD + a·D + b) straight from the registers:
    // a thread holds, for its rows, the symmetric (column tile o) and antisymmetric (column
    // tile NP1 + o') outputs of the same tiles tl, so L_ab = L⁺ + L⁻, L_ba = L⁺ − L⁻ here
    constexpr int NP1 = D * (D + 1) / 2, NH = TPC / 8;   // column tiles per output: 1 (3D), 2 (2D)
#pragma unroll
    for (int mi = 0; mi < KMI; ++mi) {
      const int rr = warp * 8 * KMI + mi * 8 + fr;   // KW warps × 8·KMI rows
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int tl = hh * 8 + 2 * fc + e;
#pragma unroll
          for (int ab = 0; ab < DD; ++ab) {
            const int a = ab / D, b = ab % D, lo = a < b ? a : b, hi = a < b ? b : a;
            const double sp = acc[mi][sym_index(D, lo, hi) * NH + hh][e];
            double v = sp;
            if (a != b) {
              const double am = acc[mi][(NP1 + anti_index(D, lo, hi)) * NH + hh][e];
#ifndef IGA_EXPERIMENT_K3_NO_STAGE_DADD   // timing only (wrong K): no FP64 add in the staging
              v = a < b ? sp + am : sp - am;
#else
              v = a < b ? sp : am;
#endif
            }
            sC[rr * K3_CROW + tl * DD + ab] = v;
          }
        }
    }
  }
  __syncthreads();
  if (EPI == 0) {   // nzdata (Eq. 58): local[row][t*DD + a*D + b]
    const int64_t N = n_tiles * DD;
    constexpr int RW = TPC * DD;   // the block's 72 columns of a row are contiguous in nzdata
    const uint64_t pol = l2_policy_evict_first();
    if (t0 + TPC <= n_tiles && (N & 1) == 0) {   // whole block, 16-B aligned rows: 16-B stores
      for (int i = tid; i < K3_BM * RW / 2; i += KT) {
        const int rr = i / (RW / 2), c = 2 * (i % (RW / 2));
        const int64_t gr = m0 + rr;
        if (gr < M) st2_hint(out + gr * N + t0 * DD + c, sC[rr * K3_CROW + c], sC[rr * K3_CROW + c + 1], pol);
      }
    } else {
      for (int i = tid; i < K3_BM * RW; i += KT) {
        const int rr = i / RW, c = i % RW, tl = c / DD, ab = c % DD;
        const int64_t gr = m0 + rr, t = t0 + tl;
        if (gr < M && t < n_tiles) out[gr * N + t * DD + ab] = sC[rr * K3_CROW + c];
      }
    }
    return;
  }
  if (EPI == 2) {
    // thread e: c1 = L u_J (diagonal: L_sym u_I) of row e and c2 = Lᵀ u_I of row tperm[e]
    // (position e of the (B, A) order).  Each run of equal A (c1) / equal B (c2) inside the
    // row block is summed into the run's partial slot in a fixed tree order: a segmented
    // suffix sum over the lanes of the warp (shuffles, every lane busy; a single thread
    // summing its run in order cost 2.1 of the apply's 15.9 ms at cfg5, sparse two-level
    // sums in shared memory 1.3 ms), and the one run per half that crosses rows 31|32 is
    // completed through shared memory after the tile loop.
    static_assert(EPI != 2 || K3_BM == 64, "apply epilogue: two warps per half, one cut at rows 31|32");
    double *xs = sC + K3_BM * K3_CROW;   // [tile of the CTA][c1 | c2][lower | upper part][D]
    const int et = tperm[m0 + er];
    const int64_t rt = m0 + et;
    const bool live = r < M, live_t = rt < M;
    const int A = live ? pairA[r] : 0, B = live ? pairB[r] : 0;
    const int At = live_t ? pairA[rt] : 0, Bt = live_t ? pairB[rt] : 0;
    const int g1 = ap.g1len[m0 + er], g2 = ap.g2len[m0 + er];   // run length | position in the run << 8
    const int len1 = g1 & 0xff, pos1 = g1 >> 8, len2 = g2 & 0xff, pos2 = g2 >> 8;
    const int wmax1 = __reduce_max_sync(0xffffffffu, len1), wmax2 = __reduce_max_sync(0xffffffffu, len2);
    // the run's rows [start, end) of the block, this warp's rows [wb, wb + 32)
    const int wb = er & ~31, st1 = er - pos1, en1 = st1 + len1, st2 = er - pos2, en2 = st2 + len2;
    const bool lead1 = len1 && er == max(st1, wb), cross1 = len1 && st1 < 32 && en1 > 32;
    const bool lead2 = len2 && er == max(st2, wb), cross2 = len2 && st2 < 32 && en2 > 32;
    // the partial slots belong to the runs' first rows
    const int64_t sl1 = pos1 == 0 ? ap.g1slot[m0 + er] : -1, sl2 = pos2 == 0 ? ap.g2slot[m0 + er] : -1;
    // u of node(t, B) (diagonal: node(t, A)) and of node(t, A_t) for all TPT tiles, from the
    // per-tile gathered copy, loaded at once (the accumulators are dead here): one L2 latency
    double uBv[TPT][D], uAv[TPT][D];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int64_t t = t0 + et0 + k < n_tiles ? t0 + et0 + k : n_tiles - 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        uBv[k][a] = live ? ap.u[(t * nl + B) * D + a] : 0.0;
        uAv[k][a] = live_t ? ap.u[(t * nl + At) * D + a] : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const int tl = et0 + k;
      const int64_t t = t0 + tl;
      const bool tv = t < n_tiles;
      double c1[D], c2[D];
#pragma unroll
      for (int a = 0; a < D; ++a) c1[a] = c2[a] = 0.0;
      if (tv && live) {
        const double *L = sC + er * K3_CROW;
        const double *uv = uBv[k];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) c1[a] += (A == B && a > b ? L[tl * DD + b * D + a] : L[tl * DD + a * D + b]) * uv[b];
      }
      if (tv && live_t && At != Bt) {
        const double *L = sC + et * K3_CROW;
        const double *uv = uAv[k];
#pragma unroll
        for (int b = 0; b < D; ++b)
#pragma unroll
          for (int a = 0; a < D; ++a) c2[b] += L[tl * DD + a * D + b] * uv[a];
      }
      // segmented suffix sums: after the steps the first lane of every (warp, run) segment
      // holds the sum of the segment's rows (steps beyond the warp's longest run are skipped)
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        if (off < wmax1) {
          const bool in = lane + off < 32 && pos1 + off < len1;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double x = __shfl_down_sync(0xffffffffu, c1[a], off);
            if (in) c1[a] += x;
          }
        }
        if (off < wmax2) {
          const bool in = lane + off < 32 && pos2 + off < len2;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double x = __shfl_down_sync(0xffffffffu, c2[a], off);
            if (in) c2[a] += x;
          }
        }
      }
      if (lead1) {
        if (cross1) {
#pragma unroll
          for (int a = 0; a < D; ++a) xs[((tl * 2 + 0) * 2 + (er >= 32)) * D + a] = c1[a];
        } else if (tv) {
#pragma unroll
          for (int a = 0; a < D; ++a) ap.part[(t * ap.P + sl1) * D + a] = c1[a];
        }
      }
      if (lead2) {
        if (cross2) {
#pragma unroll
          for (int a = 0; a < D; ++a) xs[((tl * 2 + 1) * 2 + (er >= 32)) * D + a] = c2[a];
        } else if (tv) {
#pragma unroll
          for (int a = 0; a < D; ++a) ap.part[(t * ap.P + sl2) * D + a] = c2[a];
        }
      }
    }
    __syncthreads();
    // the runs cut at rows 31|32: lower part + upper part, by the run's first row
    if (cross1 && pos1 == 0) {
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const int tl = et0 + k;
        const int64_t t = t0 + tl;
        if (t < n_tiles)
#pragma unroll
          for (int a = 0; a < D; ++a)
            ap.part[(t * ap.P + sl1) * D + a] = xs[((tl * 2 + 0) * 2 + 0) * D + a] + xs[((tl * 2 + 0) * 2 + 1) * D + a];
      }
    }
    if (cross2 && pos2 == 0) {
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const int tl = et0 + k;
        const int64_t t = t0 + tl;
        if (t < n_tiles)
#pragma unroll
          for (int a = 0; a < D; ++a)
            ap.part[(t * ap.P + sl2) * D + a] = xs[((tl * 2 + 1) * 2 + 0) * D + a] + xs[((tl * 2 + 1) * 2 + 1) * D + a];
      }
    }
    return;
  }
  // fused scatter (R9).  Pass 1: row er, blocks (I,J) (diagonal blocks mirrored from
  // their upper triangle); pass 2: row tperm[er] of the (B, A)-ordered block, blocks
  // (J,I) = Lᵀ.  Both orders put neighbouring blocks of one CSR row in neighbouring lanes;
  // the d-double row segments of a warp's 32 blocks are then stored cooperatively — lane
  // l writes words l, l+32, ... of the warp's 32·d words — so runs of adjacent blocks leave
  // as whole 32-B sectors instead of 8/16-B pieces per lane.
#if IGA_K3_CL > 1   // experiment: thread-block clusters (profiles/r02_scatter_experiments.md)
  // EPI 3 (thread-block clusters of K3_CL row blocks): the transposed pass walks the cluster's
  // K3_CL·64 rows in (B, A) order (cperm), entry q·64 + er for the CTA of cluster rank q, and
  // reads the block from the staging tile of the CTA that computed it (distributed shared
  // memory), so the (J,I) blocks of one CSR row J coming from neighbouring A leave as one run
  int et, src_rank = 0;
  int64_t rt;
  if constexpr (EPI == 3) {
    const int64_t cb = (mb / K3_CL) * (K3_CL * K3_BM);
    const int rs = cperm[cb + (mb % K3_CL) * K3_BM + er];
    rt = cb + rs;
    src_rank = rs / K3_BM;
    et = rs % K3_BM;
    cluster_arrive_release();   // this CTA's tile is staged
  } else {
    et = tperm[m0 + er];
    rt = m0 + et;
  }
  const bool live = r < M, live_t = rt < M;
  const int A = live ? pairA[r] : 0, B = live ? pairB[r] : 0;
  const int At = live_t ? pairA[rt] : 0, Bt = live_t ? pairB[rt] : 0;
  int32_t em[TPT], emt[TPT];
  int64_t riA[TPT], riB[TPT];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int64_t t = t0 + et0 + k < n_tiles ? t0 + et0 + k : n_tiles - 1;
    em[k] = live ? emap[t * M + r] : 0;
    riA[k] = live ? rowinfo[t * nl + A] : 0;
    emt[k] = live_t ? emap[t * M + rt] : 0;
    riB[k] = live_t ? rowinfo[t * nl + Bt] : 0;
  }
  // lanes hold (o = CSR offset of their block's first row segment or -1, row stride,
  // smem row | diagonal << 8); word w of the warp's row segments comes from lane w/D,
  // column w%D, and the D row segments of a block are o, o + stride, ...: one set of
  // shuffles per block serves its D rows; value L[ra][cb] of that lane's block
  auto coop = [&](int64_t o, int str, int pk, int tl, bool transposed) {
    // all shuffles, then all shared loads, then the predicated stores (CSR values are written once:
    // L2 evict-first)
    int64_t ob[D];
    int sstr[D], p[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int src = (32 * j + lane) / D;
      ob[j] = __shfl_sync(0xffffffffu, o, src);
      sstr[j] = __shfl_sync(0xffffffffu, str, src);
      p[j] = __shfl_sync(0xffffffffu, pk, src);
    }
    double v[D][D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int c = (32 * j + lane) % D, sb = p[j] & 0xff;
      const bool db = (p[j] >> 8) & 1;
#pragma unroll
      for (int idx = 0; idx < D; ++idx) {
        int ra = transposed ? c : idx, cb = transposed ? idx : c;
        if (db && ra > cb) { const int x = ra; ra = cb; cb = x; }
        if (EPI == 3 && transposed)   // the block's staging tile may live in another CTA of the cluster
          v[j][idx] = cluster_map(sC, p[j] >> 9)[sb * K3_CROW + tl * DD + ra * D + cb];
        else
          v[j][idx] = sC[sb * K3_CROW + tl * DD + ra * D + cb];
      }
    }
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS
    const uint64_t pol = l2_policy_evict_first();
#endif
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int c = (32 * j + lane) % D;
#pragma unroll
      for (int idx = 0; idx < D; ++idx)
        if (ob[j] >= 0) {
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS
          st_hint(out + ob[j] + (int64_t)idx * sstr[j] + c, v[j][idx], pol);
#else
          out[ob[j] + (int64_t)idx * sstr[j] + c] = v[j][idx];
#endif
        }
    }
  };
  auto pass1 = [&](int k) {   // row er: side slot or K(I,J) = L
    const int tl = et0 + k;
    const int32_t ev = em[k];
#ifdef IGA_EXPERIMENT_NO_SCATTER
    if (ev != 12345) return;
#endif
    if (live && ev < 0) {   // one of several contributions: side slot, summed by K4
      const double *L = sC + er * K3_CROW;
      double *o = side + (int64_t)(-ev - 1) * DD;
#pragma unroll
      for (int q = 0; q < DD; ++q) o[q] = L[tl * DD + q];
    }
    const bool w1 = live && ev >= 0 && riA[k] >= 0;   // riA < 0: row of another shard
#ifndef IGA_EXPERIMENT_K3_LINEAR
    const int64_t off1 = DD * (riA[k] >> 24) + D * (ev & 0xffff);
    const int str1 = D * (int)(riA[k] & 0xffffff);
#else   // timing only (wrong K): the same stores to contiguous blocks (scatter addresses removed)
    const int64_t off1 = ((t0 + tl) * M + r) * DD;
    const int str1 = D;
#endif
#ifndef IGA_EXPERIMENT_NO_PASS1
    coop(w1 ? off1 : -1, str1, er | (A == B ? 256 : 0), tl, false);
#endif
  };
  auto pass2 = [&](int k) {   // row rt of the (B, A) order: K(J,I) = Lᵀ
    const int tl = et0 + k;
#ifdef IGA_EXPERIMENT_NO_SCATTER
    if (em[k] != 12345) return;
#endif
    const int32_t evt = emt[k];
    const bool w2 = live_t && evt >= 0 && At != Bt && riB[k] >= 0;
#ifndef IGA_EXPERIMENT_K3_LINEAR
    const int64_t off2 = DD * (riB[k] >> 24) + D * (evt >> 16);
    const int str2 = D * (int)(riB[k] & 0xffffff);
#else
    const int64_t off2 = (n_tiles * M - 1 - ((t0 + tl) * M + rt)) * DD;
    const int str2 = D;
#endif
#ifndef IGA_EXPERIMENT_NO_PASS2
    coop(w2 ? off2 : -1, str2, et | (src_rank << 9), tl, true);
#endif
  };
  if constexpr (EPI == 3) {
    // all (I,J) blocks, then — once every tile of the cluster is staged — the pooled (J,I) pass;
    // no CTA leaves while another may still read its staging tile
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      if (t0 + et0 + k >= n_tiles) break;   // warp-uniform
      pass1(k);
    }
    cluster_wait_acquire();
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      if (t0 + et0 + k >= n_tiles) break;
      pass2(k);
    }
    cluster_arrive_release();
    cluster_wait_acquire();
  } else {
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      if (t0 + et0 + k >= n_tiles) break;   // warp-uniform
      pass1(k);
      pass2(k);
    }
  }
#else
#ifndef IGA_EXPERIMENT_K3_ROWDESC
  const int et = tperm[m0 + er];
  const int64_t rt = m0 + et;
  const bool live = r < M, live_t = rt < M;
  const int A = live ? pairA[r] : 0, B = live ? pairB[r] : 0;
  const int At = live_t ? pairA[rt] : 0, Bt = live_t ? pairB[rt] : 0;
#else   // one 16-B row descriptor {A | B << 16, At | Bt << 16, tperm, 0}: one load level less
  const int4 rd = rowdesc[m0 + er];
  const int et = rd.z;
  const int64_t rt = m0 + et;
  const bool live = rd.x >= 0, live_t = rd.y >= 0;
  const int A = live ? rd.x & 0xffff : 0, B = live ? rd.x >> 16 : 0;
  const int At = live_t ? rd.y & 0xffff : 0, Bt = live_t ? rd.y >> 16 : 0;
#endif
  int32_t em[TPT], emt[TPT];
  int64_t riA[TPT], riB[TPT];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int64_t t = t0 + et0 + k < n_tiles ? t0 + et0 + k : n_tiles - 1;
    em[k] = live ? emap[t * M + r] : 0;
    riA[k] = live ? rowinfo[t * nl + A] : 0;
    emt[k] = live_t ? emap[t * M + rt] : 0;
    riB[k] = live_t ? rowinfo[t * nl + Bt] : 0;
  }
  // cooperative row-segment stores: word w = 32j + lane of the warp's 32·D words of one row
  // index comes from the block of lane src_j = w / D (its row), column c_j = w % D.  Lanes hold
  // (o = CSR offset of their block's first row segment or -1, row stride); the shared-memory
  // offsets of every (j, idx) word are tile-independent and computed once here: pass 1 reads
  // L[idx][c] of row er(src) (diagonal rows: L[min][max], R9), pass 2 reads L[c][idx] of row
  // tperm(src) — per tile only the offsets and strides are shuffled.
#ifndef IGA_EXPERIMENT_K3_COOP_V22
  int so1[D][D], so2[D];
  {
    const bool dg = A == B;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int w = 32 * j + lane, src = w / D, c = w % D;
      const int er_s = (er & ~31) + src;                      // row of lane src (er = tid % 64)
      const int et_s = __shfl_sync(0xffffffffu, et, src);
      const bool dg_s = __shfl_sync(0xffffffffu, (int)dg, src) != 0;
#pragma unroll
      for (int idx = 0; idx < D; ++idx) {
        const int lo = dg_s && idx > c ? c : idx, hi = dg_s && idx > c ? idx : c;
        so1[j][idx] = er_s * K3_CROW + lo * D + hi;
      }
      so2[j] = et_s * K3_CROW + c * D;
    }
  }
  auto coop = [&](int64_t o, int str, int tl, bool transposed) {
    int64_t ob[D];
    int sstr[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int src = (32 * j + lane) / D;
      ob[j] = __shfl_sync(0xffffffffu, o, src);
      sstr[j] = __shfl_sync(0xffffffffu, str, src);
    }
    const double *st = sC + tl * DD;
    double v[D][D];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int idx = 0; idx < D; ++idx) v[j][idx] = transposed ? st[so2[j] + idx] : st[so1[j][idx]];
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS
    const uint64_t pol = l2_policy_evict_first();   // CSR values are written once (a constant: folded by ptxas)
#endif
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (ob[j] >= 0) {
        double *g = out + ob[j] + (32 * j + lane) % D;
#pragma unroll
        for (int idx = 0; idx < D; ++idx) {
#if defined(IGA_EXPERIMENT_K3_FULLSECTOR)   // timing only (wrong K): every store instruction writes 256 aligned bytes
#if IGA_EXPERIMENT_K3_FULLSECTOR == 1   // (I,J) pass only
          if (transposed) st_hint(g + (int64_t)idx * sstr[j], v[j][idx], pol); else
#elif IGA_EXPERIMENT_K3_FULLSECTOR == 2   // (J,I) pass only
          if (!transposed) st_hint(g + (int64_t)idx * sstr[j], v[j][idx], pol); else
#endif
          {
            const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;   // 2^30 doubles < nnz at cfg5
            const int64_t u = ((cta * 4 + warp) * 72 + ((tl - et0) * 2 + (transposed ? 1 : 0)) * 9 + j * 3 + idx) * 32;
            st_hint(out + (u & ((int64_t(1) << 30) - 1)) + lane, v[j][idx], pol);
          }
#elif defined(IGA_EXPERIMENT_K3_PASS2_EVICT_NORMAL)   // experiment: the transposed pass's partial sectors stay in L2
          if (transposed) g[(int64_t)idx * sstr[j]] = v[j][idx];
          else st_hint(g + (int64_t)idx * sstr[j], v[j][idx], pol);
#elif defined(IGA_EXPERIMENT_K3_PASS2_EVICT_LAST)
          st_hint(g + (int64_t)idx * sstr[j], v[j][idx], transposed ? l2_policy_evict_last() : pol);
#elif !defined(IGA_EXPERIMENT_K3_NO_L2_HINTS)
          st_hint(g + (int64_t)idx * sstr[j], v[j][idx], pol);
#else
          g[(int64_t)idx * sstr[j]] = v[j][idx];
#endif
        }
      }
    }
  };
#else   // the v22 cooperative store (shuffled row / diagonal flag per tile and word)
  // lanes hold (o = CSR offset of their block's first row segment or -1, row stride,
  // smem row | diagonal << 8); word w of the warp's row segments comes from lane w/D,
  // column w%D, and the D row segments of a block are o, o + stride, ...: one set of
  // shuffles per block serves its D rows; value L[ra][cb] of that lane's block
  auto coop_v22 = [&](int64_t o, int str, int pk, int tl, bool transposed) {
    // all shuffles, then all shared loads, then the predicated stores (CSR values are written once:
    // L2 evict-first)
    int64_t ob[D];
    int sstr[D], p[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int src = (32 * j + lane) / D;
      ob[j] = __shfl_sync(0xffffffffu, o, src);
      sstr[j] = __shfl_sync(0xffffffffu, str, src);
      p[j] = __shfl_sync(0xffffffffu, pk, src);
    }
    double v[D][D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int c = (32 * j + lane) % D, sb = p[j] & 0xff;
      const bool db = (p[j] >> 8) & 1;
#pragma unroll
      for (int idx = 0; idx < D; ++idx) {
        int ra = transposed ? c : idx, cb = transposed ? idx : c;
        if (db && ra > cb) { const int x = ra; ra = cb; cb = x; }
        v[j][idx] = sC[sb * K3_CROW + tl * DD + ra * D + cb];
      }
    }
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS
    const uint64_t pol = l2_policy_evict_first();
#endif
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int c = (32 * j + lane) % D;
#pragma unroll
      for (int idx = 0; idx < D; ++idx)
        if (ob[j] >= 0) {
#ifndef IGA_EXPERIMENT_K3_NO_L2_HINTS
          st_hint(out + ob[j] + (int64_t)idx * sstr[j] + c, v[j][idx], pol);
#else
          out[ob[j] + (int64_t)idx * sstr[j] + c] = v[j][idx];
#endif
        }
    }
  };
  auto coop = [&](int64_t o, int str, int tl, bool transposed) {
    coop_v22(o, str, transposed ? et : (er | (A == B ? 256 : 0)), tl, transposed);
  };
#endif
#ifdef IGA_K3_TILE_UNROLL   // experiment: unroll factor of the tile loop (default: full)
#pragma unroll K3_TILE_UNROLL
#else
#pragma unroll
#endif
  for (int k = 0; k < TPT; ++k) {
    const int tl = et0 + k;
    if (t0 + tl >= n_tiles) break;   // warp-uniform
    const int32_t ev = em[k];
#ifdef IGA_EXPERIMENT_NO_SCATTER
    if (ev != 12345) continue;
#endif
    if (live && ev < 0) {   // one of several contributions: side slot, summed by K4
      const double *L = sC + er * K3_CROW;
      double *o = side + (int64_t)(-ev - 1) * DD;
#pragma unroll
      for (int q = 0; q < DD; ++q) o[q] = L[tl * DD + q];
    }
    const bool w1 = live && ev >= 0 && riA[k] >= 0;   // riA < 0: row of another shard
#ifndef IGA_EXPERIMENT_K3_LINEAR
    const int64_t off1 = DD * (riA[k] >> 24) + D * (ev & 0xffff);
    const int str1 = D * (int)(riA[k] & 0xffffff);
#else   // timing only (wrong K): the same stores to contiguous blocks (scatter addresses removed)
    const int64_t off1 = ((t0 + tl) * M + r) * DD;
    const int str1 = D;
#endif
#ifndef IGA_EXPERIMENT_NO_PASS1
    coop(w1 ? off1 : -1, str1, tl, false);
#endif
    const int32_t evt = emt[k];
    const bool w2 = live_t && evt >= 0 && At != Bt && riB[k] >= 0;
#ifndef IGA_EXPERIMENT_K3_LINEAR
    const int64_t off2 = DD * (riB[k] >> 24) + D * (evt >> 16);
    const int str2 = D * (int)(riB[k] & 0xffffff);
#else
    const int64_t off2 = (n_tiles * M - 1 - ((t0 + tl) * M + rt)) * DD;
    const int str2 = D;
#endif
#if !defined(IGA_EXPERIMENT_NO_PASS2) && !defined(IGA_EXPERIMENT_K3_SPLIT_PASSES)
    coop(w2 ? off2 : -1, str2, tl, true);
#endif
  }
#ifdef IGA_EXPERIMENT_K3_SPLIT_PASSES   // experiment: all (I,J) blocks first, then all (J,I) blocks
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int tl = et0 + k;
    if (t0 + tl >= n_tiles) break;
    const int32_t evt = emt[k];
    const bool w2 = live_t && evt >= 0 && At != Bt && riB[k] >= 0;
    coop(w2 ? DD * (riB[k] >> 24) + D * (evt >> 16) : -1, D * (int)(riB[k] & 0xffffff), tl, true);
  }
#endif
#endif
}

#ifdef IGA_EXPERIMENT_K3P
// ---------------------------------------------------------------------------------
// K3p: the persistent, warp-specialised K3 with the fused CSR scatter (EPI 1, the hot path).
// One CTA per SM walks the 64-row × 72-column output tiles L = blockIdx.x + i·gridDim.x
// (row blocks fastest, as K3's grid).  Its 12 MMA warps form 3 groups of 4 (one warp of
// each group per SM sub-partition); group g takes the tiles i ≡ g (mod 3) through its own
// 3-stage bulk-copy ring (the last of its warps to release a stage refills it with the
// group's next chunk, across tile boundaries) — three independent rings per SM, like three
// co-resident K3 CTAs, so the groups drift apart in phase and the DMMA pipe does not wait
// on one hand-off.  At the end of a tile a group stages it in shared memory (L_t[a][b], as
// K3) into staging slot i % 2 and goes on with its next tile; 8 store warps scatter the
// staged tiles in the order i (K3's cooperative CSR row-segment stores, side slots for
// shared blocks), with the maps of the next tile loaded while they wait for it.  Register
// split by setmaxnreg: MMA warpgroups 128 registers per thread, store warpgroups 64.
// Hand-off per slot: mbarriers `slot_full` (the 128 threads of a group) and `slot_free`
// (the 256 store threads); tiles are handed off in the order i.
constexpr int K3P_GROUPS = 3, K3P_GW = 4;                            // MMA groups, warps per group
constexpr int K3P_MMA_WARPS = K3P_GROUPS * K3P_GW, K3P_STORE_WARPS = 8;
constexpr int K3P_THREADS = 32 * (K3P_MMA_WARPS + K3P_STORE_WARPS);
constexpr int K3P_MMA_REGS = 120, K3P_STORE_REGS = 56;
static_assert(K3P_MMA_WARPS % 4 == 0 && K3P_STORE_WARPS % 4 == 0, "setmaxnreg acts per warpgroup");
// setmaxnreg only redistributes the CTA's launch allocation (65536 / threads, rounded down to 8)
static_assert(K3P_MMA_WARPS * K3P_MMA_REGS + K3P_STORE_WARPS * K3P_STORE_REGS <=
                  (K3P_MMA_WARPS + K3P_STORE_WARPS) * (65536 / K3P_THREADS / 8 * 8), "register file");
constexpr int K3P_BM = 16 * K3P_GW;                                  // 64 rows = one FM row block
constexpr int K3P_STAGES = 3, K3P_SLOTS = 2;
constexpr int K3P_A_CHUNK = K3P_BM * BK, K3P_B_CHUNK = BN * BK;     // doubles
constexpr int K3P_STAGE = K3P_A_CHUNK + K3P_B_CHUNK;
constexpr size_t K3P_RING = sizeof(double) * (size_t)K3P_GROUPS * K3P_STAGES * K3P_STAGE;
constexpr size_t K3P_STAGING = sizeof(double) * (size_t)K3P_SLOTS * K3P_BM * K3_CROW;
constexpr size_t K3P_OFF_BAR = K3P_RING + K3P_STAGING;
constexpr int K3P_BATCHES = 4;                                       // ring of fetched tile batches
constexpr size_t K3P_SMEM = K3P_OFF_BAR + (K3P_GROUPS * K3P_STAGES + 2 * K3P_SLOTS) * sizeof(uint64_t) +
                            (K3P_GROUPS * K3P_STAGES + 2 * K3P_BATCHES) * sizeof(int);
static_assert(K3P_BM == IGA_K3_BM, "a K3p tile is one 64-row FM row block (tperm is per 64-row block)");
static_assert(K3P_SMEM <= 227 * 1024, "K3p shared memory");

// what a store warp needs of one (row half, tile) unit, loaded ahead of the staged tile
template <int SPT>
struct K3pUnits {
  int A[2], B[2], At[2], Bt[2], et[2];
  int32_t em[2][SPT], emt[2][SPT];
  int64_t riA[2][SPT], riB[2][SPT];
};

// Dynamic tile scheduling: the CTA takes its tiles in batches of K3P_GROUPS consecutive tiles
// from a global counter (items 3b, 3b+1, 3b+2 of the CTA = tiles L0, L0+1, L0+2), so that
// all SMs work on neighbouring tiles at any time (as the hardware block scheduler would):
// the CSR rows of a tile are then written within a short window and merge in L2, and the
// table and coefficient chunks stay L2-resident.  Batch b lives in slot b % 4 of a smem
// ring; whoever needs it first claims the slot (it held batch b-4, which nobody needs any
// more: the store warps are at most ~7 items behind the groups) and fetches it.
__device__ __forceinline__ int k3p_batch(int b, int *bseq, int *bL, int *ctr) {
  volatile int *vs = bseq, *vl = bL;
  const int slot = b % K3P_BATCHES;
  for (;;) {
    const int cur = vs[slot];
    if (cur == b) {
      __threadfence_block();
      return vl[slot];
    }
    if (cur == b - K3P_BATCHES && atomicCAS(&bseq[slot], cur, -(1 << 30) - b) == cur) {   // claim and fetch
      const int L0 = atomicAdd(ctr, K3P_GROUPS);
      vl[slot] = L0;
      __threadfence_block();
      atomicExch(&bseq[slot], b);
      return L0;
    }
    __nanosleep(32);
  }
}

template <int D>
__global__ void __launch_bounds__(K3P_THREADS, 1)
k3p_contract(const double *__restrict__ tabA, const double *__restrict__ coef, int nkc, int ksteps, int ksplit,
             int64_t M, int n_mb, int n_work, int64_t n_tiles, double *__restrict__ out,
             const int32_t *__restrict__ pairA, const int32_t *__restrict__ pairB, const int32_t *__restrict__ emap,
             const int64_t *__restrict__ rowinfo, int nl, double *__restrict__ side,
             const int4 *__restrict__ rowdesc, int *__restrict__ work_ctr) {
  constexpr int DD = D * D, TPC = D == 3 ? 8 : 16, NE = D == 3 ? 9 : 8;
  constexpr int NP1 = D * (D + 1) / 2, NH = TPC / 8, SPT = TPC / K3P_STORE_WARPS;
  extern __shared__ __align__(128) double smem[];
  double *staging = smem + K3P_RING / sizeof(double);
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + K3P_OFF_BAR);  // [group][stage]
  uint64_t *slot_full = full + K3P_GROUPS * K3P_STAGES, *slot_free = slot_full + K3P_SLOTS;
  int *released = reinterpret_cast<int *>(slot_free + K3P_SLOTS);                           // [group][stage]
  int *bseq = released + K3P_GROUPS * K3P_STAGES, *bL = bseq + K3P_BATCHES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tile of the CTA's item i (-1: none left); one lane asks, the warp shares the answer
  auto tile_of = [&](int i) -> int {
    int L = 0;
    if (lane == 0) {
      L = k3p_batch(i / K3P_GROUPS, bseq, bL, work_ctr) + i % K3P_GROUPS;
      if (L >= n_work) L = -1;
    }
    return __shfl_sync(0xffffffffu, L, 0);
  };
  if (tid == 0) {
    for (int b = 0; b < K3P_BATCHES; ++b) bseq[b] = b - K3P_BATCHES;   // "holds batch b-4": free
    for (int s = 0; s < K3P_GROUPS * K3P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    for (int s = 0; s < K3P_SLOTS; ++s) {
      mbar_init(&slot_full[s], 32 * K3P_GW);
      mbar_init(&slot_free[s], 32 * K3P_STORE_WARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp < K3P_MMA_WARPS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(K3P_MMA_REGS));
    // ---------------- MMA group grp: rows [16·lw, 16·lw + 16) of its tiles i ≡ grp (mod 3) ----
    const int grp = warp / K3P_GW, lw = warp % K3P_GW;
    double *sA = smem + grp * K3P_STAGES * K3P_STAGE;
    uint64_t *gfull = full + grp * K3P_STAGES;
    int *grel = released + grp * K3P_STAGES;
    // operand chunk 0 of a tile L
    auto bases = [&](int L, const double *&ga, const double *&gb) {
      const int mb = L % n_mb, nb = L / n_mb;
      ga = tabA + (int64_t)mb * nkc * K3P_A_CHUNK;
      gb = coef + (int64_t)nb * nkc * K3P_B_CHUNK;
    };
    auto produce = [&](const double *ga, const double *gb, int kc, int st) {
      double *a = sA + st * K3P_STAGE;
      mbar_expect_tx(&gfull[st], (uint32_t)(K3P_STAGE * 8));
      bulk_g2s(a, ga + (int64_t)kc * K3P_A_CHUNK, K3P_A_CHUNK * 8, &gfull[st]);
      bulk_g2s(a + K3P_A_CHUNK, gb + (int64_t)kc * K3P_B_CHUNK, K3P_B_CHUNK * 8, &gfull[st]);
    };
    // the group's k-th item is i = grp + 3k; the ring runs K3P_STAGES chunks ahead: (pk, pkc)
    int pk = 0, pkc = 0;
    const double *pga = nullptr, *pgb = nullptr;
    int pL = tile_of(grp);
    if (pL >= 0) bases(pL, pga, pgb);
    for (int st = 0; st < K3P_STAGES && pL >= 0; ++st) {   // prologue: the first K3P_STAGES chunks
      if (warp % K3P_GW == 0 && lane == 0) produce(pga, pgb, pkc, st);
      if (++pkc == nkc) {
        pkc = 0;
        ++pk;
        pL = tile_of(grp + K3P_GROUPS * pk);
        if (pL >= 0) bases(pL, pga, pgb);
      }
    }
    const int fr = lane >> 2, fc = lane & 3;
    int st = 0;
    uint32_t ph = 0;
    for (int k = 0;; ++k) {
      const int i = grp + K3P_GROUPS * k;
      const int L = tile_of(i);
      if (L < 0) break;
      const int mb = L % n_mb;
      const int64_t wr0 = (int64_t)mb * K3P_BM + lw * 16;
      const int nmi = wr0 >= M ? 0 : (wr0 + 8 < M ? 2 : 1);
      double acc[MI][NI][2];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      for (int kc = 0; kc < nkc; ++kc) {
        mbar_wait(&gfull[st], ph);
        const double *a_st = sA + st * K3P_STAGE, *b_st = a_st + K3P_A_CHUNK;
        const int s0 = kc * (BK / 4), ns = min(BK / 4, ksteps - s0), jj = max(0, min(ksplit - s0, ns));
        if (nmi == 2) k3_chunk<2, NE>(a_st, b_st, lw * 2, lane, ns, jj, acc);
        else if (nmi == 1) k3_chunk<1, NE>(a_st, b_st, lw * 2, lane, ns, jj, acc);
        __syncwarp();
        if (lane == 0) {   // the last warp of the group to release a stage refills it
          __threadfence_block();
          if (atomicAdd(&grel[st], 1) == K3P_GW - 1) {
            grel[st] = 0;
            __threadfence_block();
            if (pL >= 0) produce(pga, pgb, pkc, st);
          }
        }
        if (++pkc == nkc) {
          pkc = 0;
          ++pk;
          if (pL >= 0) {
            pL = tile_of(grp + K3P_GROUPS * pk);
            if (pL >= 0) bases(pL, pga, pgb);
          }
        }
        if (++st == K3P_STAGES) { st = 0; ph ^= 1u; }
      }
      // hand the tile to the store warps through staging slot i % 2, in the order i: first
      // item i-1 must have been handed off (its slot_full phase; a parity wait is exact here
      // because this group itself handed off i-3 on that slot), then the store warps must be
      // done with item i-2 (slot_free; they finished i-4 before i-2 could be handed off)
      const int slot = i % K3P_SLOTS;
      if (i >= 1) mbar_wait(&slot_full[(i - 1) % K3P_SLOTS], (uint32_t)(((i - 1) / K3P_SLOTS) & 1));
      if (i >= K3P_SLOTS) mbar_wait(&slot_free[slot], (uint32_t)((i / K3P_SLOTS - 1) & 1));
      double *sC = staging + slot * (K3P_BM * K3_CROW);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int rr = lw * 16 + mi * 8 + fr;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int tl = hh * 8 + 2 * fc + e;
#pragma unroll
            for (int ab = 0; ab < DD; ++ab) {
              const int a = ab / D, b = ab % D, lo = a < b ? a : b, hi = a < b ? b : a;
              const double sp = acc[mi][sym_index(D, lo, hi) * NH + hh][e];
              double v = sp;
              if (a != b) {
                const double am = acc[mi][(NP1 + anti_index(D, lo, hi)) * NH + hh][e];
                v = a < b ? sp + am : sp - am;
              }
              sC[rr * K3_CROW + tl * DD + ab] = v;
            }
          }
      }
      mbar_arrive(&slot_full[slot]);
    }
    return;
  }
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(K3P_STORE_REGS));
  // ---------------- store warps: tiles tl = sw + 8k of every tile item, both 32-row halves ----
  const int sw = warp - K3P_MMA_WARPS;
  auto load_item = [&](int L, K3pUnits<SPT> &u) {
    const int mb = L % n_mb, nb = L / n_mb;
    const int64_t m0 = (int64_t)mb * K3P_BM, t0 = (int64_t)nb * TPC;
#pragma unroll
    for (int h = 0; h < 2; ++h) {   // one 16-byte descriptor per row: no dependent load chain
      const int e = h * 32 + lane;
      const int4 q = rowdesc[m0 + e];
      u.et[h] = q.z;
      u.A[h] = q.x < 0 ? -1 : (q.x & 0xffff);
      u.B[h] = q.x < 0 ? 0 : (q.x >> 16);
      u.At[h] = q.y < 0 ? -1 : (q.y & 0xffff);
      u.Bt[h] = q.y < 0 ? 0 : (q.y >> 16);
      const int64_t r = m0 + e, rt = m0 + q.z;
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        const int64_t t = min(t0 + sw + K3P_STORE_WARPS * k, n_tiles - 1);
        u.em[h][k] = q.x >= 0 ? emap[t * M + r] : 0;
        u.riA[h][k] = q.x >= 0 ? rowinfo[t * nl + u.A[h]] : 0;
        u.emt[h][k] = q.y >= 0 ? emap[t * M + rt] : 0;
        u.riB[h][k] = q.y >= 0 ? rowinfo[t * nl + u.Bt[h]] : 0;
      }
    }
  };
  // warm L2 with the epilogue map rows of a later tile (emap is streamed once from HBM)
  auto prefetch_item = [&](int L) {
    const int mb = L % n_mb, nb = L / n_mb;
    const int64_t t = (int64_t)nb * TPC + sw + K3P_STORE_WARPS * (lane >> 1);
    if (lane < 2 * SPT && t < n_tiles) prefetch_l2(emap + t * M + (int64_t)mb * K3P_BM + 32 * (lane & 1));
  };
  K3pUnits<SPT> u;
  int L = tile_of(0);
  if (L >= 0) load_item(L, u);
  {
    const int L1 = tile_of(1);
    if (L1 >= 0) prefetch_item(L1);
  }
  for (int i = 0; L >= 0; ++i) {
    const int nb = L / n_mb;
    const int64_t t0 = (int64_t)nb * TPC;
    const int slot = i % K3P_SLOTS;
    const double *sC = staging + slot * (K3P_BM * K3_CROW);
    auto coop = [&](int64_t o, int str, int pk, int tl, bool transposed) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int w = 32 * j + lane, src = w / D, c = w - src * D;
        const int64_t ob = __shfl_sync(0xffffffffu, o, src);
        const int sstr = __shfl_sync(0xffffffffu, str, src);
        const int p = __shfl_sync(0xffffffffu, pk, src);
        if (ob >= 0) {
          const int sb = p & 0xff;
          const bool db = (p >> 8) & 1;
#pragma unroll
          for (int idx = 0; idx < D; ++idx) {
            int ra = transposed ? c : idx, cb = transposed ? idx : c;
            if (db && ra > cb) { const int x = ra; ra = cb; cb = x; }
            out[ob + (int64_t)idx * sstr + c] = sC[sb * K3_CROW + tl * DD + ra * D + cb];
          }
        }
      }
    };
    mbar_wait(&slot_full[slot], (uint32_t)((i / K3P_SLOTS) & 1));
#ifndef IGA_EXPERIMENT_K3P_NO_STORE   // (timing only, wrong K: the main loop and the hand-off without the scatter)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = h * 32 + lane;
      const bool live = u.A[h] >= 0, live_t = u.At[h] >= 0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        const int tl = sw + K3P_STORE_WARPS * k;
        if (t0 + tl >= n_tiles) break;   // warp-uniform
        const int32_t ev = u.em[h][k];
        if (live && ev < 0) {   // one of several contributions: side slot, summed by K4
          const double *Lr = sC + e * K3_CROW + tl * DD;
          double *o = side + (int64_t)(-ev - 1) * DD;
#pragma unroll
          for (int q = 0; q < DD; ++q) o[q] = Lr[q];
        }
        const int64_t ri = u.riA[h][k];
        const bool w1 = live && ev >= 0 && ri >= 0;   // ri < 0: row of another shard
        coop(w1 ? DD * (ri >> 24) + D * (ev & 0xffff) : -1, D * (int)(ri & 0xffffff),
             e | (u.A[h] == u.B[h] ? 256 : 0), tl, false);
        const int32_t evt = u.emt[h][k];
        const int64_t rj = u.riB[h][k];
        const bool w2 = live_t && evt >= 0 && u.At[h] != u.Bt[h] && rj >= 0;
        coop(w2 ? DD * (rj >> 24) + D * (evt >> 16) : -1, D * (int)(rj & 0xffffff), u.et[h], tl, true);
      }
    }
#endif
    mbar_arrive(&slot_free[slot]);
    L = tile_of(i + 1);
    if (L >= 0) {
      load_item(L, u);   // in flight while the next tile is computed / staged
      const int L2 = tile_of(i + 2);
      if (L2 >= 0) prefetch_item(L2);
    }
  }
}

template <int D>
static cudaError_t launch_k3p(const Handle &h, double *out, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k3p_contract<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3P_SMEM);
  if (e) return e;
  int dev = 0, nsm = 148;
  if ((e = cudaGetDevice(&dev)) || (e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
  const int64_t n_mb = h.Mpad / K3P_BM;
  const int64_t n_work = n_mb * (h.Npad / BN);
  if (n_work >= (1ll << 31)) return cudaErrorInvalidConfiguration;
  const unsigned grid = (unsigned)std::min<int64_t>((n_work + K3P_GROUPS - 1) / K3P_GROUPS, nsm);
  if ((e = cudaMemsetAsync(h.d_flag + 3, 0, sizeof(int), s))) return e;   // the tile counter (d_flag[3])
  k3p_contract<D><<<grid, K3P_THREADS, K3P_SMEM, s>>>(h.d_tabA, h.d_coef, h.ks3 / BK, h.k3_steps, h.k3_split, h.M,
                                                      (int)n_mb, (int)n_work, h.n_tiles, out, h.d_pairA, h.d_pairB,
                                                      h.d_emap, h.d_rowinfo, h.n_local_ctrl, h.d_side, h.d_rowdesc,
                                                      h.d_flag + 3);
  return cudaGetLastError();
}

#endif  // IGA_EXPERIMENT_K3P

template <int D, int EPI>
static cudaError_t launch_k3(const Handle &h, double *out, cudaStream_t s, ApplyArgs ap = ApplyArgs{}) {
  cudaError_t e = cudaFuncSetAttribute(k3_contract<D, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3_smem<EPI>());
  if (e) return e;
  dim3 grid((unsigned)(h.Mpad / K3_BM), (unsigned)(h.Npad / BN));   // M-blocks fastest
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  if (EPI == 3) {   // thread-block clusters of K3_CL row blocks
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(K3Cfg<EPI>::THREADS);
    cfg.dynamicSmemBytes = k3_smem<EPI>();
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K3_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k3_contract<D, EPI>, h.d_tabA, h.d_coef, (int)(h.ks3 / BK), h.k3_steps, h.k3_split,
                              h.M, h.n_tiles, out, h.d_pairA, h.d_pairB, h.d_emap, h.d_rowinfo, h.n_local_ctrl,
                              h.d_side, h.d_tperm, h.d_cperm, h.d_rowdesc, ap);
  }
  k3_contract<D, EPI><<<grid, K3Cfg<EPI>::THREADS, k3_smem<EPI>(), s>>>(h.d_tabA, h.d_coef, h.ks3 / BK, h.k3_steps, h.k3_split, h.M,
                                                        h.n_tiles, out, h.d_pairA, h.d_pairB, h.d_emap, h.d_rowinfo,
                                                        h.n_local_ctrl, h.d_side, h.d_tperm, h.d_cperm, h.d_rowdesc, ap);
  return cudaGetLastError();
}

// y[i] = Σ over the (tile, A) occurrences of owned node i (fixed order) of Σ over A's
// partial slots (fixed order): deterministic, no atomics
template <int D>
__global__ void __launch_bounds__(256)
k4_apply_gather(const double *__restrict__ part, int64_t P, const int32_t *__restrict__ sA_ptr,
                const int32_t *__restrict__ sA_slot, const int64_t *__restrict__ inv_ptr,
                const int32_t *__restrict__ inv_ent, int nl, int64_t n_nodes, double *__restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  double acc[D];
#pragma unroll
  for (int a = 0; a < D; ++a) acc[a] = 0.0;
  for (int64_t f = inv_ptr[i]; f < inv_ptr[i + 1]; ++f) {
    const int32_t e = inv_ent[f];
    const int64_t t = e / nl;
    const int A = e % nl;
    for (int q = sA_ptr[A]; q < sA_ptr[A + 1]; ++q) {
      const double *src = part + (t * P + sA_slot[q]) * D;
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += src[a];
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) y[i * D + a] = acc[a];
}

// ug[t][A][a] = u[node(t, A)·d + a]: u gathered per tile once, so the apply epilogue reads it
// without the node-map indirection
template <int D>
__global__ void k3_gather_u(const double *__restrict__ u, const int32_t *__restrict__ node_map, int64_t n,
                            double *__restrict__ ug) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t I = node_map[i];
#pragma unroll
  for (int a = 0; a < D; ++a) ug[i * D + a] = u[I * D + a];
}

cudaError_t launch_apply(const Handle &h, const double *u, double *y, cudaStream_t s) {
  const int64_t n = h.n_tiles * h.n_local_ctrl;
  double *ug = h.d_ug;
  if (h.d == 2) k3_gather_u<2><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(u, h.d_node_map, n, ug);
  else k3_gather_u<3><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(u, h.d_node_map, n, ug);
  ApplyArgs ap{ug, h.d_part, h.P, h.d_g1len, h.d_g2len, h.d_g1slot, h.d_g2slot, h.d_node_map};
  cudaError_t e = h.d == 2 ? launch_k3<2, 2>(h, nullptr, s, ap) : launch_k3<3, 2>(h, nullptr, s, ap);
  if (e) return e;
  const unsigned blocks = (unsigned)((h.n_nodes + 255) / 256);
  if (h.d == 2)
    k4_apply_gather<2><<<blocks, 256, 0, s>>>(h.d_part, h.P, h.d_sA_ptr, h.d_sA_slot, h.d_inv_ptr, h.d_inv_ent,
                                              h.n_local_ctrl, h.n_nodes, y);
  else
    k4_apply_gather<3><<<blocks, 256, 0, s>>>(h.d_part, h.P, h.d_sA_ptr, h.d_sA_slot, h.d_inv_ptr, h.d_inv_ent,
                                              h.n_local_ctrl, h.n_nodes, y);
  return cudaGetLastError();
}

cudaError_t launch_contraction(const Handle &h, double *vals, double *local, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
#ifdef IGA_EXPERIMENT_K3P   // the persistent warp-specialised K3 (profiles/r02_k3p_experiment.md)
  if (vals) e = h.d == 2 ? launch_k3p<2>(h, vals, s) : launch_k3p<3>(h, vals, s);
#else
#if IGA_K3_CL > 1   // experiment: thread-block clusters (profiles/r02_scatter_experiments.md)
  if (vals) e = h.d == 2 ? launch_k3<2, 3>(h, vals, s) : launch_k3<3, 3>(h, vals, s);
#else
  if (vals) e = h.d == 2 ? launch_k3<2, 1>(h, vals, s) : launch_k3<3, 1>(h, vals, s);
#endif
#endif
  if (e) return e;
  if (local) e = h.d == 2 ? launch_k3<2, 0>(h, local, s) : launch_k3<3, 0>(h, local, s);
  return e;
}

// ---------------------------------------------------------------------------------
// K5a.  X (the coefficient of every local entry in uᵀK^πv, R9/R13) is generated by a
// memory-bound kernel into the fragment-major B-operand layout, then contracted with
// the table by a two-operand bulk-copy DMMA GEMM.  Generating X inside the GEMM costs
// more: its DMUL/DFMA share the FP64 datapath with DMMA and starve behind it
// (measured: 27.9 ms vs 22.7 ms for the GEMM alone at cfg5, profiles/r01_*).

// X̃[col][n] for the tile patch of grid.x and the 72 columns of N-block grid.y in the
// sym layout of the Eq. 38-reduced contraction: block column n = o·TPC + tl
// holds X̃⁺ = X_aa or X_ab + X_ba (o < n_p1: symmetric output (a,b), a <= b) or
// X̃⁻ = X_ab − X_ba (antisymmetric output a < b), X_ab the coefficient of L[a][b] in uᵀK^πv
// (R9/R13; diagonal rows: X_ab = u_a v_b + u_b v_a for a < b, u_a v_a for a = b, 0 for
// a > b).  Chunk kc of the patch is written as one contiguous FM chunk (coalesced).
// Thread (warp w, lane) owns row k = 4w + lane%4 of every chunk and the 9 columns
// n_j = 8j + lane/4, i.e. FM elements e = 128j + 32w + lane: one pair per chunk, the
// per-column offsets are loop invariants.
template <int D>
__global__ void __launch_bounds__(128)
k5x_gen(const int32_t *__restrict__ k5_pair, const int32_t *__restrict__ pinfo, const int32_t *__restrict__ node_map,
        int nl, const double *__restrict__ u, const double *__restrict__ v, int64_t n_tiles, int nkc,
        double *__restrict__ X) {
  constexpr int TPC = D == 3 ? 8 : 16, NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2;
  extern __shared__ __align__(128) double smem[];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int64_t nb = blockIdx.y, t0 = nb * TPC;
  const int kc0 = pinfo[3 * p], kc1 = pinfo[3 * (p + 1)], off = pinfo[3 * p + 1], nc = pinfo[3 * p + 2];
  // per-tile stride nc·D + 1 (odd): the 8 tiles a warp reads at once fall in distinct banks
  const int ts = nc * D + 1;
  double *us = smem, *vs = smem + TPC * ts;
  for (int i = tid; i < TPC * nc; i += 128) {
    const int tl = i / nc, A = i % nc;
    const int64_t t = t0 + tl;
    double *uo = us + tl * ts + A * D, *vo = vs + tl * ts + A * D;
    if (t < n_tiles) {
      const int64_t I = node_map[t * nl + off + A];
#pragma unroll
      for (int a = 0; a < D; ++a) { uo[a] = u[I * D + a]; vo[a] = v[I * D + a]; }
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) { uo[a] = 0.0; vo[a] = 0.0; }
    }
  }
  const int k = 4 * (tid >> 5) + (lane & 3);
  // column tile j holds output o = j (3D) or j/2 (2D), (a, b) and the mode are compile-time
  // constants; the thread's tile(s) tl are fixed: 3D one tile (lane/4), 2D two (lane/4, +8)
  constexpr int NTL = D == 3 ? 1 : 2;
  int toff[NTL];
#pragma unroll
  for (int it = 0; it < NTL; ++it) toff[it] = (it * 8 + (lane >> 2)) * ts;
  __syncthreads();
  int32_t pr = k5_pair[(int64_t)kc0 * BK + k];
  for (int kc = kc0; kc < kc1; ++kc) {
    const int32_t pr_next = kc + 1 < kc1 ? k5_pair[(int64_t)(kc + 1) * BK + k] : -1;
    double *dst = X + (nb * nkc + kc) * (int64_t)K5_X_CHUNK_ + tid;
    double x[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) x[j] = 0.0;
    if (pr >= 0) {
      const int A = (pr & 0xffff) * D, B = (pr >> 16) * D;
      double uA[NTL][D], vA[NTL][D], uB[NTL][D], vB[NTL][D];
#pragma unroll
      for (int it = 0; it < NTL; ++it)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          uA[it][c] = us[toff[it] + A + c];
          vA[it][c] = vs[toff[it] + A + c];
          uB[it][c] = us[toff[it] + B + c];
          vB[it][c] = vs[toff[it] + B + c];
        }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int o = D == 3 ? j : j >> 1, it = D == 3 ? 0 : (j & 1);
        if (o >= NP1 + NP2) continue;                               // unused column (2D)
        int a = 0, b = 0;
        if (o < NP1) sym_pair(D, o, a, b);
        else anti_pair(D, o - NP1, a, b);
        // X_ab = u_{I,a} v_{J,b} + u_{J,b} v_{I,a} (K5x's original arithmetic)
        const double xab = fma(uB[it][b], vA[it][a], uA[it][a] * vB[it][b]);
        if (o < D) x[j] = A == B ? 0.5 * xab : xab;                 // X_aa
        else if (A == B) x[j] = xab;                                 // diagonal row: X_ba = 0 (a < b)
        else {
          const double xba = fma(uB[it][a], vA[it][b], uA[it][b] * vB[it][a]);
          x[j] = o < NP1 ? xab + xba : xab - xba;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) dst[128 * j] = x[j];
    pr = pr_next;
  }
}

#ifndef IGA_K5_STAGES
#define IGA_K5_STAGES 4
#endif
constexpr int K5_STAGES = IGA_K5_STAGES;
constexpr int K5_A_CHUNK = BM * BK, K5_B_CHUNK = BN * BK;   // doubles
constexpr int K5_WP = BM + 1;                                // W staging pitch
constexpr int K5_THREADS = 32 * N_MMA_WARPS;
constexpr size_t K5_OFF_BAR = sizeof(double) * (size_t)K5_STAGES * (K5_A_CHUNK + K5_B_CHUNK);
constexpr size_t K5_SMEM = K5_OFF_BAR + K5_STAGES * (sizeof(uint64_t) + sizeof(int));
static_assert(sizeof(double) * BN * K5_WP <= K5_OFF_BAR, "W staging must fit in the stages");

// Y[n][κ] = Σ_col tabAT[κ][col] X̃[col][n]: CTA = 128 κ rows × 72 columns, 8 MMA warps of
// 16×72; the last MMA warp to release a stage refills it.  Eq. 38-reduced:
// κ rows of part 1 (< k5s) meet the symmetric columns (tiles [0, 6)), part 2 rows
// (< k5k) the antisymmetric ones ([6, NE)); no DMMA for the other pairings or padding.
template <int D, bool SPLIT>
__global__ void __launch_bounds__(K5_THREADS, 1)
k5a_wgemm(const double *__restrict__ tabAT, const double *__restrict__ X, int nkc, int64_t N,
          double *__restrict__ Wout, int ldw, const uint8_t *__restrict__ k5_mode) {
  constexpr int NE = D == 3 ? 9 : 8;
  extern __shared__ __align__(128) double smem[];
  double *sA = smem, *sB = smem + K5_STAGES * K5_A_CHUNK;
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + K5_OFF_BAR);
  int *released = reinterpret_cast<int *>(full + K5_STAGES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t kb = blockIdx.x, nb = blockIdx.y;
  // split-K for small problems (too few N-blocks to fill the SMs): segment z of the reduction
  // writes its own partial Y, summed in segment order by k5a_reduce
  const double *gA = tabAT + kb * (int64_t)nkc * K5_A_CHUNK, *gB = X + nb * (int64_t)nkc * K5_B_CHUNK;
  if (SPLIT) {
    const int kc_lo = (int)((int64_t)blockIdx.z * nkc / gridDim.z);
    const int kc_hi = (int)((int64_t)(blockIdx.z + 1) * nkc / gridDim.z);
    gA += (int64_t)kc_lo * K5_A_CHUNK;
    gB += (int64_t)kc_lo * K5_B_CHUNK;
    nkc = kc_hi - kc_lo;
    Wout += (int64_t)blockIdx.z * N * ldw;
  }
  // part (1, 2; 0 = padding) of each of the warp's two 8-row groups: part(mi0)·3 + part(mi1)
  // (host-balanced placement of the κ groups, Handle::k5_gphys)
  const int mode = k5_mode[kb * N_MMA_WARPS + warp];
  if (tid == 0) {
    for (int s = 0; s < K5_STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto produce = [&](int kc) {   // the last MMA warp to release a stage refills it
    const int st = kc % K5_STAGES;
    mbar_expect_tx(&full[st], (K5_A_CHUNK + K5_B_CHUNK) * 8);
    bulk_g2s(sA + st * K5_A_CHUNK, gA + (int64_t)kc * K5_A_CHUNK, K5_A_CHUNK * 8, &full[st]);
    bulk_g2s(sB + st * K5_B_CHUNK, gB + (int64_t)kc * K5_B_CHUNK, K5_B_CHUNK * 8, &full[st]);
  };
  if (tid == 0)
    for (int s = 0; s < K5_STAGES && s < nkc; ++s) produce(s);
  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int kc = 0; kc < nkc; ++kc) {
    const int st = kc % K5_STAGES;
    mbar_wait(&full[st], (kc / K5_STAGES) & 1);
    const double *a_st = sA + st * K5_A_CHUNK, *b_st = sB + st * K5_B_CHUNK;
    switch (mode) {
      case 4: mma_steps<4, 0, 2, 0, 6>(a_st, b_st, warp * MI, lane, 0, acc); break;    // (1, 1)
      case 8: mma_steps<4, 0, 2, 6, NE>(a_st, b_st, warp * MI, lane, 0, acc); break;   // (2, 2)
      case 5:                                                                          // (1, 2)
        mma_steps<4, 0, 1, 0, 6>(a_st, b_st, warp * MI, lane, 0, acc);
        mma_steps<4, 1, 1, 6, NE>(a_st, b_st, warp * MI, lane, 0, acc);
        break;
      case 3: mma_steps<4, 0, 1, 0, 6>(a_st, b_st, warp * MI, lane, 0, acc); break;    // (1, pad)
      case 6: mma_steps<4, 0, 1, 6, NE>(a_st, b_st, warp * MI, lane, 0, acc); break;   // (2, pad)
      default: break;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&released[st], 1) == N_MMA_WARPS - 1) {
        released[st] = 0;
        __threadfence_block();
        if (kc + K5_STAGES < nkc) produce(kc + K5_STAGES);
      }
    }
  }
  __syncthreads();   // all stages consumed: stage W[n][κ] in shared memory
  double *sW = smem;
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int kap = warp * 16 + mi * 8 + fr, n = ni * 8 + 2 * fc;
      sW[n * K5_WP + kap] = acc[mi][ni][0];
      sW[(n + 1) * K5_WP + kap] = acc[mi][ni][1];
    }
  __syncthreads();
  for (int i = tid; i < BN * BM; i += K5_THREADS) {
    const int n = i / BM, kap = i % BM;
    const int64_t gn = nb * BN + n, gk = kb * BM + kap;
    if (gn < N && gk < ldw) Wout[gn * ldw + gk] = sW[n * K5_WP + kap];
  }
}

// ---------------------------------------------------------------------------------
// K5g: K5x fused into K5a.  Besides the 16 MMA warps, 4 generator warps build every B
// chunk (X̃, K5x's arithmetic and thread mapping) in shared memory from u, v staged per tile
// patch, so X̃ never goes to HBM.  Per stage: fullA (the TMA'd table chunk), fullB (the 128
// generator threads), emptyB (the last MMA warp to release a stage lets the generators
// refill it).  Every MMA warp keeps only the accumulators of its κ-group parts (registers:
// the 640-thread CTA must fit 65,536).
#ifndef IGA_K5G_GEN_WARPS
#define IGA_K5G_GEN_WARPS 12   // three groups of 4 warps take chunks in turn (8: 13.55 ms, 12: 13.40, 16: 13.63)
#endif
constexpr int K5G_GEN_WARPS = IGA_K5G_GEN_WARPS;
static_assert(K5G_GEN_WARPS % 4 == 0, "generator groups of 4 warps (128 threads per chunk)");
static_assert(K5G_GEN_WARPS / 4 <= 3, "the generators' emptyB parity wait needs groups <= X̃ stages (SB >= 3)");
constexpr int K5G_THREADS = 32 * (N_MMA_WARPS + K5G_GEN_WARPS);

struct K5gArgs {
  const double *tabAT;
  const int32_t *k5_pair, *pinfo, *node_map;
  int nl, n_patches;
  const double *u, *v;
  int64_t n_tiles;
  int nkc;          // chunks of the whole reduction (Kp / 16)
  int64_t N;        // Y rows (N-blocks × 72)
  double *Wout;
  int ldw;
  const uint8_t *k5_mode;
  int ts;           // per-tile stride of the u/v staging (max_patch_ctrl·D + 1)
  const int32_t *k5_extra;   // modes 11/12: the extra single-column piece (local group | column << 16)
};

// SA table stages (TMA, refilled by the last MMA warp to release one) and SB >= SA X̃ stages
// (written by the generators, released by every MMA warp's arrival): the generators run up to
// SB chunks ahead of the MMA warps, so a chunk whose FP64 products were throttled behind the
// DMMAs is still ready in time
template <int SA, int SB>
struct K5gSmem {
  static constexpr size_t STAGES = sizeof(double) * ((size_t)SA * K5_A_CHUNK + (size_t)SB * K5_B_CHUNK);
  static size_t bytes(int d, int ts) {
    return STAGES + sizeof(double) * 2 * (size_t)(d == 3 ? 8 : 16) * ts + (SA + 2 * SB) * sizeof(uint64_t) +
           SA * sizeof(int);
  }
};

template <int LO0, int HI0, int LO1, int HI1>
struct K5gAcc {
  static constexpr int N0 = HI0 - LO0, N1 = HI1 - LO1;
  double a0[N0 > 0 ? N0 : 1][2], a1[N1 > 0 ? N1 : 1][2];
};

template <int D, int SA, int SB, int LO0, int HI0, int LO1, int HI1, bool HX = false>
__device__ __forceinline__ void k5g_mma_role(const K5gArgs &g, double *smem, int kc_lo, int nkc, int warp, int lane,
                                             const double *gA, int xg = 0, int xn = 0) {
  constexpr int N0 = HI0 - LO0, N1 = HI1 - LO1;
  double *sA = smem, *sB = smem + SA * K5_A_CHUNK;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + K5gSmem<SA, SB>::STAGES +
                                                 sizeof(double) * 2 * (D == 3 ? 8 : 16) * g.ts);
  uint64_t *fullB = fullA + SA, *emptyB = fullB + SB;
  int *released = reinterpret_cast<int *>(emptyB + SB);
  K5gAcc<LO0, HI0, LO1, HI1> acc;
  double accx0 = 0.0, accx1 = 0.0;   // HX: the extra piece (group xg, column tile xn)
#pragma unroll
  for (int i = 0; i < (N0 > 0 ? N0 : 1); ++i) acc.a0[i][0] = acc.a0[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < (N1 > 0 ? N1 : 1); ++i) acc.a1[i][0] = acc.a1[i][1] = 0.0;
  const int g0 = warp * 2;
  for (int kc = 0; kc < nkc; ++kc) {
    const int st = kc % SA, sb = kc % SB;
    mbar_wait(&fullA[st], (kc / SA) & 1);
    mbar_wait(&fullB[sb], (kc / SB) & 1);
    const double *a_st = sA + st * K5_A_CHUNK, *b_st = sB + sb * K5_B_CHUNK;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double a0 = 0.0, a1 = 0.0, b[NI];
      if (N0 > 0) a0 = a_st[(g0 * 4 + kk) * 32 + lane];
      if (N1 > 0) a1 = a_st[((g0 + 1) * 4 + kk) * 32 + lane];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        if ((ni >= LO0 && ni < HI0) || (ni >= LO1 && ni < HI1)) b[ni] = b_st[(ni * 4 + kk) * 32 + lane];
#pragma unroll
      for (int ni = LO0; ni < HI0; ++ni) dmma884(acc.a0[ni - LO0][0], acc.a0[ni - LO0][1], a0, b[ni]);
#pragma unroll
      for (int ni = LO1; ni < HI1; ++ni) dmma884(acc.a1[ni - LO1][0], acc.a1[ni - LO1][1], a1, b[ni]);
      if (HX) dmma884(accx0, accx1, a_st[(xg * 4 + kk) * 32 + lane], b_st[(xn * 4 + kk) * 32 + lane]);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&emptyB[sb]);   // this warp is done with the X̃ stage (release: its reads come first)
      __threadfence_block();
      if (atomicAdd(&released[st], 1) == N_MMA_WARPS - 1) {
        released[st] = 0;
        __threadfence_block();
        if (kc + SA < nkc) {   // refill the table chunk by TMA
#ifdef IGA_EXPERIMENT_K5G_NO_TABLE_REFILL   // timing only (wrong g): the first SA table chunks are reused
          mbar_arrive(&fullA[st]);
#else
          mbar_expect_tx(&fullA[st], K5_A_CHUNK * 8);
          bulk_g2s(sA + st * K5_A_CHUNK, gA + (int64_t)(kc + SA) * K5_A_CHUNK, K5_A_CHUNK * 8, &fullA[st]);
#endif
        }
      }
    }
  }
  named_bar(1, K5G_THREADS);   // all stages consumed (generators included): stage Y in smem
  double *sW = smem;
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int ni = LO0; ni < HI0; ++ni) {
    const int kap = warp * 16 + fr, n = ni * 8 + 2 * fc;
    sW[n * K5_WP + kap] = acc.a0[ni - LO0][0];
    sW[(n + 1) * K5_WP + kap] = acc.a0[ni - LO0][1];
  }
#pragma unroll
  for (int ni = LO1; ni < HI1; ++ni) {
    const int kap = warp * 16 + 8 + fr, n = ni * 8 + 2 * fc;
    sW[n * K5_WP + kap] = acc.a1[ni - LO1][0];
    sW[(n + 1) * K5_WP + kap] = acc.a1[ni - LO1][1];
  }
  if (HX) {
    const int kap = xg * 8 + fr, n = xn * 8 + 2 * fc;
    sW[n * K5_WP + kap] = accx0;
    sW[(n + 1) * K5_WP + kap] = accx1;
  }
}

template <int D, int SA, int SB>
__device__ __forceinline__ void k5g_gen_role(const K5gArgs &g, double *smem, int kc_lo, int nkc, int64_t nb, int gtid) {
  constexpr int TPC = D == 3 ? 8 : 16, NP1 = D * (D + 1) / 2, NP2 = D * (D - 1) / 2, NTL = D == 3 ? 1 : 2;
  constexpr int NG = K5G_GEN_WARPS / 4;          // groups of 4 warps: one chunk per group at a time
  constexpr int NGT = 32 * K5G_GEN_WARPS;
  double *sB = smem + SA * K5_A_CHUNK;
  double *us = smem + K5gSmem<SA, SB>::STAGES / sizeof(double), *vs = us + TPC * g.ts;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(vs + TPC * g.ts);
  uint64_t *fullB = fullA + SA, *emptyB = fullB + SB;
  const int grp = gtid >> 7, gt = gtid & 127;
  const int lane = gt & 31, k = 4 * (gt >> 5) + (lane & 3);
  const int64_t t0 = nb * TPC;
  const int kc_hi = kc_lo + nkc;
  int toff[NTL];
#pragma unroll
  for (int it = 0; it < NTL; ++it) toff[it] = (it * 8 + (lane >> 2)) * g.ts;
  // the tile patches overlapping this CTA's chunk range, in order; all groups walk the same
  // sequence (so the per-patch barriers match), group grp takes chunks c0 + grp, c0 + grp + NG, ...
  int p = 0;
  while (p + 1 < g.n_patches && g.pinfo[3 * (p + 1)] <= kc_lo) ++p;
  for (; p < g.n_patches && g.pinfo[3 * p] < kc_hi; ++p) {
    const int c0 = max(g.pinfo[3 * p], kc_lo), c1 = min(g.pinfo[3 * (p + 1)], kc_hi);
    const int off = g.pinfo[3 * p + 1], nc = g.pinfo[3 * p + 2];
#ifdef IGA_EXPERIMENT_K5G_STAGE_ONCE
    if (c0 == kc_lo) {   // timing experiment only: stage the first patch once
#else
    {   // restage u, v of the patch's control points for the CTA's tiles
#endif
      named_bar(2, NGT);   // every group is done with the previous patch's u, v
      for (int i = gtid; i < TPC * nc; i += NGT) {
        const int tl = i / nc, A = i % nc;
        const int64_t t = t0 + tl;
        double *uo = us + tl * g.ts + A * D, *vo = vs + tl * g.ts + A * D;
        if (t < g.n_tiles) {
          const int64_t I = g.node_map[t * g.nl + off + A];
#pragma unroll
          for (int a = 0; a < D; ++a) { uo[a] = g.u[I * D + a]; vo[a] = g.v[I * D + a]; }
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) { uo[a] = 0.0; vo[a] = 0.0; }
        }
      }
      named_bar(2, NGT);
    }
    // the pair index of the group's next chunk is loaded one chunk ahead
    int32_t prn = c0 + grp < c1 ? g.k5_pair[(int64_t)(c0 + grp) * BK + k] : -1;
    for (int gkc = c0 + grp; gkc < c1; gkc += NG) {
      const int32_t pr = prn;
      prn = gkc + NG < c1 ? g.k5_pair[(int64_t)(gkc + NG) * BK + k] : -1;
      const int kc = gkc - kc_lo, st = kc % SB;
      if (kc >= SB) mbar_wait(&emptyB[st], ((kc / SB) - 1) & 1);
      double x[NI];
#pragma unroll
      for (int j = 0; j < NI; ++j) x[j] = 0.0;
      if (pr >= 0) {
        const int A = (pr & 0xffff) * D, B = (pr >> 16) * D;
        double uA[NTL][D], vA[NTL][D], uB[NTL][D], vB[NTL][D];
#pragma unroll
        for (int it = 0; it < NTL; ++it)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            uA[it][c] = us[toff[it] + A + c];
            vA[it][c] = vs[toff[it] + A + c];
            uB[it][c] = us[toff[it] + B + c];
            vB[it][c] = vs[toff[it] + B + c];
          }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int o = D == 3 ? j : j >> 1, it = D == 3 ? 0 : (j & 1);
          if (o >= NP1 + NP2) continue;
          int a = 0, b = 0;
          if (o < NP1) sym_pair(D, o, a, b);
          else anti_pair(D, o - NP1, a, b);
#ifdef IGA_EXPERIMENT_K5G_NO_GEN_MATH   // timing only (wrong g): no FP64 arithmetic in the generators
          x[j] = uB[it][b] + vA[it][a];
          continue;
#endif
          const double xab = fma(uB[it][b], vA[it][a], uA[it][a] * vB[it][b]);
          if (o < D) x[j] = A == B ? 0.5 * xab : xab;
          else if (A == B) x[j] = xab;
          else {
            const double xba = fma(uB[it][a], vA[it][b], uA[it][b] * vB[it][a]);
            x[j] = o < NP1 ? xab + xba : xab - xba;
          }
        }
      }
      double *dst = sB + st * K5_B_CHUNK + gt;
#pragma unroll
      for (int j = 0; j < NI; ++j) dst[128 * j] = x[j];
      __syncwarp();   // the warp's stores happen before its elected arrival (release)
      if (lane == 0) mbar_arrive(&fullB[st]);
    }
  }
  named_bar(1, K5G_THREADS);
}

template <int D, int SA, int SB, bool SPLIT>
__global__ void __launch_bounds__(K5G_THREADS, 1)
k5g_wgemm(const __grid_constant__ K5gArgs g) {
  constexpr int NE = D == 3 ? 9 : 8;
  static_assert(SB >= SA, "X̃ stages >= table stages");
  extern __shared__ __align__(128) double smem[];
  uint64_t *fullA = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + K5gSmem<SA, SB>::STAGES +
                                                 sizeof(double) * 2 * (D == 3 ? 8 : 16) * g.ts);
  uint64_t *fullB = fullA + SA, *emptyB = fullB + SB;
  int *released = reinterpret_cast<int *>(emptyB + SB);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t kb = blockIdx.x, nb = blockIdx.y;
  int nkc = g.nkc, kc_lo = 0;
  double *Wout = g.Wout;
  if (SPLIT) {
    kc_lo = (int)((int64_t)blockIdx.z * g.nkc / gridDim.z);
    nkc = (int)((int64_t)(blockIdx.z + 1) * g.nkc / gridDim.z) - kc_lo;
    Wout += (int64_t)blockIdx.z * g.N * g.ldw;
  }
  const double *gA = g.tabAT + (kb * (int64_t)g.nkc + kc_lo) * K5_A_CHUNK;
  if (tid == 0) {
    for (int st = 0; st < SA; ++st) {
      mbar_init(&fullA[st], 1);
      released[st] = 0;
    }
    for (int st = 0; st < SB; ++st) {
      mbar_init(&fullB[st], 4);              // the 4 warps of the group generating the chunk
      mbar_init(&emptyB[st], N_MMA_WARPS);   // every MMA warp releases the X̃ stage
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int st = 0; st < SA && st < nkc; ++st) {
      mbar_expect_tx(&fullA[st], K5_A_CHUNK * 8);
      bulk_g2s(smem + st * K5_A_CHUNK, gA + (int64_t)st * K5_A_CHUNK, K5_A_CHUNK * 8, &fullA[st]);
    }
  if (warp >= N_MMA_WARPS) {
    k5g_gen_role<D, SA, SB>(g, smem, kc_lo, nkc, nb, tid - 32 * N_MMA_WARPS);
  } else {
    switch (g.k5_mode[kb * N_MMA_WARPS + warp]) {   // parts of the warp's two κ groups
      case 4: k5g_mma_role<D, SA, SB, 0, 6, 0, 6>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 8: k5g_mma_role<D, SA, SB, 6, NE, 6, NE>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 5: k5g_mma_role<D, SA, SB, 0, 6, 6, NE>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 3: k5g_mma_role<D, SA, SB, 0, 6, 0, 0>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 6: k5g_mma_role<D, SA, SB, 6, NE, 0, 0>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      // column split (host_build.cpp, 3D): part-1 group cut to columns 0-3; extra column pieces
      case 9: k5g_mma_role<D, SA, SB, 0, 4, 0, 6>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 10: k5g_mma_role<D, SA, SB, 0, 4, 6, NE>(g, smem, kc_lo, nkc, warp, lane, gA); break;
      case 11: {
        const int x = g.k5_extra[kb * N_MMA_WARPS + warp];
        k5g_mma_role<D, SA, SB, 6, NE, 6, NE, true>(g, smem, kc_lo, nkc, warp, lane, gA, x & 0xffff, x >> 16);
        break;
      }
      case 12: {
        const int x = g.k5_extra[kb * N_MMA_WARPS + warp];
        k5g_mma_role<D, SA, SB, 0, 6, 6, NE, true>(g, smem, kc_lo, nkc, warp, lane, gA, x & 0xffff, x >> 16);
        break;
      }
      default: k5g_mma_role<D, SA, SB, 0, 0, 0, 0>(g, smem, kc_lo, nkc, warp, lane, gA); break;
    }
  }
  __syncthreads();
  const double *sW = smem;
  for (int i = tid; i < BN * BM; i += K5G_THREADS) {
    const int n = i / BM, kap = i % BM;
    const int64_t gn = nb * BN + n, gk = kb * BM + kap;
    if (gn < g.N && gk < g.ldw) Wout[gn * g.ldw + gk] = sW[n * K5_WP + kap];
  }
}

size_t k5x_smem_bytes(int d, int max_patch_ctrl) {
  return sizeof(double) * (size_t)2 * (d == 3 ? 8 : 16) * (max_patch_ctrl * d + 1);
}

template <int D>
static cudaError_t launch_k5x(const Handle &h, const double *u, const double *v, cudaStream_t s) {
  const size_t smem = k5x_smem_bytes(D, h.max_patch_ctrl);
  cudaError_t e = cudaFuncSetAttribute(k5x_gen<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  // the sensitivity runs over the owned tiles (the first n_tiles_own local tiles)
  dim3 grid((unsigned)h.n_patches, (unsigned)((h.n_tiles_own + h.tpc - 1) / h.tpc));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  k5x_gen<D><<<grid, 128, smem, s>>>(h.d_k5_pair, h.d_patch_info, h.d_node_map, h.n_local_ctrl, u, v, h.n_tiles_own,
                                     (int)(h.Kp / BK), h.d_X);
  return cudaGetLastError();
}

cudaError_t launch_sens_X(const Handle &h, const double *u, const double *v, cudaStream_t s) {
  return h.d == 2 ? launch_k5x<2>(h, u, v, s) : launch_k5x<3>(h, u, v, s);
}

// Y = Σ_z partial_z in segment order (deterministic)
__global__ void k5a_reduce(const double *__restrict__ part, int nseg, int64_t n, double *__restrict__ Y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = part[i];
  for (int z = 1; z < nseg; ++z) acc += part[(int64_t)z * n + i];
  Y[i] = acc;
}

template <int D>
static cudaError_t launch_k5a(const Handle &h, double *W, cudaStream_t s) {
  for (int32_t x : h.k5_extra)   // the K5g column split (modes 9-12) has no K5a instance
    if (x >= 0) return cudaErrorNotSupported;
  const bool split = h.k5_nseg > 1;
  cudaError_t e = cudaFuncSetAttribute(split ? k5a_wgemm<D, true> : k5a_wgemm<D, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K5_SMEM);
  if (e) return e;
  const int64_t nblk = (h.n_tiles_own + h.tpc - 1) / h.tpc;   // N-blocks of the owned tiles
  const int nseg = h.k5_nseg;
  dim3 grid((unsigned)(h.k5_rows / BM), (unsigned)nblk, (unsigned)nseg);
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  double *out = nseg > 1 ? h.d_Wpart : W;
  if (split)
    k5a_wgemm<D, true><<<grid, K5_THREADS, K5_SMEM, s>>>(h.d_tabAT, h.d_X, (int)(h.Kp / BK), nblk * BN, out,
                                                         (int)h.k5_rows, h.d_k5_mode);
  else
    k5a_wgemm<D, false><<<grid, K5_THREADS, K5_SMEM, s>>>(h.d_tabAT, h.d_X, (int)(h.Kp / BK), nblk * BN, out,
                                                          (int)h.k5_rows, h.d_k5_mode);
  if ((e = cudaGetLastError())) return e;
  if (nseg > 1) {
    const int64_t n = nblk * BN * h.k5_rows;
    k5a_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.d_Wpart, nseg, n, W);
  }
  return cudaGetLastError();
}

template <int D, int SA, int SB>
static cudaError_t launch_k5g_s(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s) {
  const int ts = h.max_patch_ctrl * D + 1;
  const size_t smem = K5gSmem<SA, SB>::bytes(D, ts);
  // the Y staging (after the main loop) overlays the stage rings and the u/v staging, not
  // the mbarriers behind them
  if (sizeof(double) * BN * K5_WP > K5gSmem<SA, SB>::STAGES + sizeof(double) * 2 * (D == 3 ? 8 : 16) * (size_t)ts)
    return cudaErrorNotSupported;
  const int64_t nblk = (h.n_tiles_own + h.tpc - 1) / h.tpc;
  const int nseg = h.k5_nseg;
  K5gArgs g{h.d_tabAT, h.d_k5_pair, h.d_patch_info, h.d_node_map, h.n_local_ctrl, h.n_patches, u, v, h.n_tiles_own,
            (int)(h.Kp / BK), nblk * BN, nseg > 1 ? h.d_Wpart : W, (int)h.k5_rows, h.d_k5_mode, ts, h.d_k5_extra};
  dim3 grid((unsigned)(h.k5_rows / BM), (unsigned)nblk, (unsigned)nseg);
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  cudaError_t e;
  if (nseg > 1) {
    if ((e = cudaFuncSetAttribute(k5g_wgemm<D, SA, SB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    k5g_wgemm<D, SA, SB, true><<<grid, K5G_THREADS, smem, s>>>(g);
  } else {
    if ((e = cudaFuncSetAttribute(k5g_wgemm<D, SA, SB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    k5g_wgemm<D, SA, SB, false><<<grid, K5G_THREADS, smem, s>>>(g);
  }
  if ((e = cudaGetLastError())) return e;
  if (nseg > 1) {
    const int64_t n = nblk * BN * h.k5_rows;
    k5a_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.d_Wpart, nseg, n, W);
  }
  return cudaGetLastError();
}

// K5x fused into K5a (X̃ generated in shared memory); cudaErrorNotSupported when the
// per-patch u, v staging does not fit beside a 3-stage ring (the caller then runs K5x + K5a)
bool sens_xw_fits(const Handle &h) {
  const int ts = h.max_patch_ctrl * h.d + 1;
  const size_t uv = sizeof(double) * 2 * (h.d == 3 ? 8 : 16) * (size_t)ts;
  const size_t lim = 227 * 1024;
  auto ok = [&](size_t stages, size_t bytes) { return bytes <= lim && sizeof(double) * BN * K5_WP <= stages + uv; };
  return ok(K5gSmem<3, 3>::STAGES, K5gSmem<3, 3>::bytes(h.d, ts));   // the smallest variant launch_sens_XW tries
}

// K5g ring shapes, first that fits: (table stages, X̃ stages)
#ifndef IGA_K5G_SB
#define IGA_K5G_SB 8   // X̃ stages of the preferred shape (cfg5: 12.94 ms; 6: 12.95, 4: 13.10, one 4-stage ring 13.13)
#endif
#ifndef IGA_K5G_SA
#define IGA_K5G_SA 3   // table stages of the preferred shape
#endif
template <int D>
static cudaError_t launch_k5g_pick(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s) {
  const int ts = h.max_patch_ctrl * D + 1;
  const size_t lim = 227 * 1024, uv = sizeof(double) * 2 * (D == 3 ? 8 : 16) * (size_t)ts;
  auto fits = [&](size_t stages, size_t bytes) { return bytes <= lim && sizeof(double) * BN * K5_WP <= stages + uv; };
#define IGA_K5G_TRY(SA_, SB_) \
  if (fits(K5gSmem<SA_, SB_>::STAGES, K5gSmem<SA_, SB_>::bytes(D, ts))) return launch_k5g_s<D, SA_, SB_>(h, u, v, W, s);
  IGA_K5G_TRY(IGA_K5G_SA, IGA_K5G_SB)
  IGA_K5G_TRY(3, 6)
  IGA_K5G_TRY(4, 4)
  IGA_K5G_TRY(3, 4)
  IGA_K5G_TRY(3, 3)
#undef IGA_K5G_TRY
  return cudaErrorNotSupported;
}

cudaError_t launch_sens_XW(const Handle &h, const double *u, const double *v, double *W, cudaStream_t s) {
  return h.d == 3 ? launch_k5g_pick<3>(h, u, v, W, s) : launch_k5g_pick<2>(h, u, v, W, s);
}

cudaError_t launch_sens_W(const Handle &h, double *W, cudaStream_t s) {
  return h.d == 2 ? launch_k5a<2>(h, W, s) : launch_k5a<3>(h, W, s);
}

}  // namespace iga
