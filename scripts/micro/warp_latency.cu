// Dependent-chain latencies (cycles per step) of the warp primitives the
// walkers put on their per-request chains, measured on one warp with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o warp_latency warp_latency.cu
#include <cstdio>
#include <cstdint>
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kIters = 4096;

__global__ void bench(unsigned seed, unsigned* out, long long* cyc) {
  __shared__ unsigned sm[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 2654435761u) & 1023u;
  __syncwarp();
  unsigned v = seed + lane;
  long long t0, t1;
  // 0: integer max (ALU), 1: redux.min, 2: ballot + ffs, 3: shfl.idx, 4: lds, 5: redux+ballot+ffs
#define CHAIN(ID, EXPR)                                            \
  t0 = clock64();                                                  \
  for (int i = 0; i < kIters; ++i) { EXPR; }                       \
  t1 = clock64();                                                  \
  if (lane == 0) cyc[ID] = t1 - t0;
  CHAIN(0, v = max(v, (unsigned)i) + 1u)
  CHAIN(1, v = __reduce_min_sync(FULL, v + lane))
  CHAIN(2, v = __ffs(__ballot_sync(FULL, ((v + lane) & 3u) == 0u)) + v)
  CHAIN(3, v = __shfl_sync(FULL, v, v & 31u) + 1u)
  CHAIN(4, v = sm[v & 1023u])
  CHAIN(5, { unsigned m = __reduce_min_sync(FULL, v + lane); v = __ffs(__ballot_sync(FULL, v + lane == m)) + m; })
  out[lane] = v;
}

int main() {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 32 * 4);
  cudaMallocManaged(&cyc, 8 * 8);
  bench<<<1, 32>>>(1u, out, cyc);
  cudaDeviceSynchronize();
  bench<<<1, 32>>>(2u, out, cyc);
  cudaDeviceSynchronize();
  const char* names[] = {"imax+add (2 ALU)", "redux.min", "ballot+ffs+add", "shfl.idx+add", "lds", "redux+ballot+ffs+add"};
  for (int k = 0; k < 6; ++k) printf("%-24s %.1f cycles/step\n", names[k], (double)cyc[k] / kIters);
  return 0;
}
