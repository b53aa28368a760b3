// Microbenchmark: latency of a dependent L2 load chain in the last CTA of a
// streaming kernel (the fold tail of the SDR kernels), with and without a
// preceding write stream. nvcc -gencode arch=compute_100a,code=sm_100a -O3 tail_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k(double* buf, size_t n_stream, const int* chain, int hops, unsigned* ctr, unsigned long long* out,
                  int mode) {
  // phase 1: stream (mode & 1: writes; mode & 2: reads)
  size_t per = n_stream / gridDim.x;
  double acc = 0;
  double* p = buf + blockIdx.x * per;
  for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
    if (mode & 2) acc += __ldcs(p + i);
    if (mode & 1) p[i] = (double)i;
  }
  if (acc == 12345.0) buf[0] = acc;
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    unsigned long long t0 = gtime();
    int idx = 0;
    for (int h = 0; h < hops; ++h) idx = __ldcg(chain + idx);
    unsigned long long t1 = gtime();
    idx += 0;
    int idx2 = 0;
    for (int h = 0; h < hops; ++h) idx2 = chain[idx2 + 0];
    unsigned long long t2 = gtime();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = idx + idx2;
    *ctr = 0;
  }
}

int main() {
  const size_t n_stream = size_t(1) << 21;  // 16.7 MB doubles
  double* buf;
  int* chain;
  unsigned* ctr;
  unsigned long long* out;
  cudaMalloc(&buf, n_stream * 8 * 4);
  const int hops = 64;
  int hchain[4096];
  for (int i = 0; i < 4096; ++i) hchain[i] = (i * 97 + 13) % 4096 / 64 * 64;  // spread
  cudaMalloc(&chain, sizeof(hchain));
  cudaMemcpy(chain, hchain, sizeof(hchain), cudaMemcpyHostToDevice);
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  cudaMallocManaged(&out, 64);
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {148, 296}) {
      for (int rep = 0; rep < 3; ++rep) {
        k<<<grid, 512>>>(buf, mode ? n_stream * (mode == 3 ? 1 : 2) : 0, chain, hops, ctr, out, mode);
        cudaDeviceSynchronize();
      }
      printf("mode %d (1=write 2=read 3=both) grid %d: ld.cg hop %.0f ns, ld hop %.0f ns\n", mode, grid,
             (double)out[0] / hops, (double)out[1] / hops);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
