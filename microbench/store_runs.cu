// store_runs.cu — how fast can B200 write FP64 data in runs of R contiguous doubles at
// scattered positions?  The K3 CSR scatter writes the 3×3 blocks of K as d-double row
// segments (24 B) that join into runs when neighbouring blocks of one CSR row are written by
// one warp instruction (profiles/r02_scatter_experiments.md).  Here every warp stores runs of
// R doubles (8·R bytes) starting at pseudo-random 8-B-aligned offsets of a large buffer, the
// words of the runs packed over the lanes exactly as K3's cooperative store packs them (lane l
// writes words l, l+32, ... of the warp's runs).  Reported per R: GB/s of useful bytes and runs
// per second; ncu gives the L2 write requests.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_runs store_runs.cu
//   ./store_runs            (prints one JSON line per run length)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {   // splitmix64
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// every warp: `iters` rounds of 32·3 words = (96 / R) runs of R doubles (R divides 96)
__global__ void __launch_bounds__(256) runs_kernel(double *out, uint64_t n_words, int R, int iters, uint64_t seed,
                                                   int align) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int runs = 96 / R;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int w = 32 * j + lane, run = w / R, c = w % R;
      const uint64_t base = mix(seed ^ ((warp * iters + it) * 97 + run)) % (n_words - R) / align * align;
      out[base + c] = (double)w;
    }
  }
  (void)runs;
}

// "slab" pattern (closer to the CSR scatter): the buffer is tiled by runs of R doubles; round
// `it` of all warps covers one slab of total_warps·(96/R) consecutive runs, every run written
// exactly once, its position inside the slab permuted (i → i·P mod S, P prime) — neighbouring
// runs come from different warps at about the same time, and a slab (~7 MB) stays in L2;
// "shifted": the same runs one double later (a run of 4k doubles then covers partial sectors)
__global__ void __launch_bounds__(256) slab_kernel(double *out, int R, int iters, int shift) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t runs = 96 / R, S = nw * runs;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int w = 32 * j + lane, run = w / R, c = w % R;
      const uint64_t i = warp * runs + run, phys = (i * 1000003ull) % S;
      out[((uint64_t)it * S + phys) * R + c + shift] = (double)w;
    }
}

// the same words, contiguous per warp (the no-scatter reference)
__global__ void __launch_bounds__(256) linear_kernel(double *out, uint64_t n_words, int iters) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint64_t base = ((warp * iters + it) * 96) % (n_words - 96);
      out[base + 32 * j + lane] = (double)lane;
    }
}

int main() {
  const uint64_t n_words = (uint64_t)3 << 29;   // 12 GB of doubles
  double *buf = nullptr;
  if (cudaMalloc(&buf, n_words * 8) != cudaSuccess) { printf("{\"error\": \"cudaMalloc\"}\n"); return 1; }
  cudaMemset(buf, 0, n_words * 8);
  const int blocks = 148 * 8, threads = 256, iters = 256;
  const double words = (double)blocks * threads / 32 * iters * 96;   // words stored per launch
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { const char *name; int R, align; };
  const Case cases[] = {{"contiguous", 96, 0},   {"random 8B-aligned", 1, 1},  {"random 8B-aligned", 2, 1},
                        {"random 8B-aligned", 3, 1},  {"random 8B-aligned", 6, 1},  {"random 8B-aligned", 12, 1},
                        {"random 8B-aligned", 24, 1}, {"random 8B-aligned", 48, 1}, {"random 8B-aligned", 96, 1},
                        {"random 32B-aligned", 4, 4}, {"random 32B-aligned", 8, 4}, {"random 32B-aligned", 16, 4},
                        {"random 32B-aligned", 32, 4}, {"random 32B-aligned", 96, 4},
                        {"slab", 1, -1}, {"slab", 2, -1}, {"slab", 3, -1}, {"slab", 6, -1}, {"slab", 12, -1},
                        {"slab", 24, -1}, {"slab", 48, -1}, {"slab", 96, -1},
                        {"slab shifted 8 B", 4, -2}, {"slab shifted 8 B", 12, -2}, {"slab shifted 8 B", 24, -2},
                        {"slab shifted 8 B", 96, -2}};
  for (int pass = 0; pass < 2; ++pass)
    for (const Case &cs : cases) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (cs.align == 0) linear_kernel<<<blocks, threads>>>(buf, n_words, iters);
        else if (cs.align < 0) slab_kernel<<<blocks, threads>>>(buf, cs.R, iters, cs.align == -2 ? 1 : 0);
        else runs_kernel<<<blocks, threads>>>(buf, n_words, cs.R, iters, 1234567ull + rep, cs.align);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      if (pass == 1)
        printf("{\"pattern\": \"%s\", \"run_doubles\": %d, \"run_bytes\": %d, \"ms\": %.4f, \"GBps\": %.1f, "
               "\"Gruns_per_s\": %.2f}\n",
               cs.name, cs.R, 8 * cs.R, best, words * 8 / (best * 1e-3) / 1e9, words / cs.R / (best * 1e-3) / 1e9);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
  cudaFree(buf);
  return 0;
}
