// Feasibility probe: one launch doing K2s(j-1) (w_j = c0 y_{j-1} + c1 w_{j-1}
// + c2 w_{j-2}, ||w_j||^2, Gram, sparse-sign S w_j) and K1(j) (y_j = A w_j
// with w_j formed on the fly at every stencil column, ||y_j||^2, window dots)
// at C5 size (512^3, SELL-DIA, 7 diagonals). Against K1 alone (the
// production loop structure) for calibration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o fused_step fused_step.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));           \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

constexpr int kSlice = 32;
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kPhi64 = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct Args {
  const double* vals;
  const int32_t* doff;
  int64_t nrows, nslices, ext_len;
  const double* Y;   // y_{j-1}
  const double* W1;  // w_{j-1}
  const double* W2;  // w_{j-2}
  double* Wout;      // w_j
  double* Ynew;      // y_j
  double c0, c1, c2;
  double* partials;  // [6][G]
  double* skp;       // [G][s]
  uint64_t key;
  int s;
};

template <int FMT, int PAIRS, bool SK>
__global__ void __launch_bounds__(64 * PAIRS) k_fused(Args a) {
  extern __shared__ __align__(16) double smem[];
  const int s = a.s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = warp >> 1, c = warp & 1;
  double* bins = smem + static_cast<int64_t>(p) * s * 32;  // [s][32] per pair
  double* xbuf = smem + static_cast<int64_t>(PAIRS) * s * 32 + p * 128;  // [2 stage][2 warp][32]
  if (SK)
    for (int i = threadIdx.x; i < PAIRS * s * 32; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();
  const double c0 = a.c0, c1 = a.c1, c2 = a.c2;
  // lane bin bases of this warp's four blocks (15 rows each at s = 120)
  uint32_t rbB[4];
  int bsz[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int l = 4 * c + e;
    const int b0 = (l * s) / 8;
    bsz[e] = ((l + 1) * s) / 8 - b0;
    rbB[e] = smem_addr(bins + b0 * 32 + lane);
  }
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t gp = static_cast<int64_t>(blockIdx.x) * PAIRS + p;
  const int64_t npairs = static_cast<int64_t>(gridDim.x) * PAIRS;
  const int64_t nq = (a.nslices + 1) / 2;
  int nx_off = 0;
  if (gp < nq && lane < FMT) {
    const int64_t sl = 2 * gp + c;
    nx_off = sl < a.nslices ? __ldg(a.doff + sl * FMT + lane) : 0;
  }
  // previous iteration's values awaiting the scatter
  double wprev[2] = {0.0, 0.0};
  int64_t qprev = -1;
  int stage = 0;
  auto scatter = [&](int64_t q, const double (&wv)[2]) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int64_t row = (2 * q + h2) * kSlice + lane;
      const uint64_t h = mix64(a.key + (static_cast<uint64_t>(row) * 2u + static_cast<uint64_t>(c) + 1u) * kPhi64);
      const uint32_t nwhi = static_cast<uint32_t>(__double2hiint(wv[h2])) ^ 0x80000000u;
      const int wlo = __double2loint(wv[h2]);
      const uint32_t hw[2] = {static_cast<uint32_t>(h), static_cast<uint32_t>(h >> 32)};
      uint32_t addr[4];
      double sv[4], tv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t f = hw[e >> 1] >> (16 * (e & 1));
        const uint32_t xb = (f & 0xFFFEu) * 15u;
        addr[e] = rbB[e] + ((xb >> 16) << 8);
        sv[e] = __hiloint2double(static_cast<int>(nwhi ^ (f << 31)), wlo);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(tv[e]) : "r"(addr[e]));
#pragma unroll
      for (int e = 0; e < 4; ++e) asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr[e]), "d"(tv[e] + sv[e]) : "memory");
    }
  };
  for (int64_t q = gp; q < nq; q += npairs) {
    const int64_t sl = 2 * q + c;
    const bool slive = sl < a.nslices;
    const int cur_off = nx_off;
    if (q + npairs < nq && lane < FMT) {
      const int64_t sn = 2 * (q + npairs) + c;
      nx_off = sn < a.nslices ? __ldg(a.doff + sn * FMT + lane) : 0;
    }
    const int64_t row = sl * kSlice + lane;
    const bool live = slive && row < a.nrows;
    // ---- all loads of the slice
    double v[FMT], xy[FMT], x1[FMT], x2[FMT];
    const double* vp = a.vals + (slive ? sl : 0) * kSlice * FMT + lane;
#pragma unroll
    for (int k = 0; k < FMT; ++k) {
      const int o = __shfl_sync(0xffffffffu, cur_off, k);
      int64_t cidx = row + o;
      cidx = cidx < 0 ? 0 : (cidx >= a.ext_len ? a.ext_len - 1 : cidx);
      v[k] = slive ? __ldcs(vp + k * kSlice) : 0.0;
      xy[k] = __ldg(a.Y + cidx);
      x1[k] = __ldg(a.W1 + cidx);
      x2[k] = __ldg(a.W2 + cidx);
    }
    const int64_t rr = live ? row : 0;
    const double oy = __ldg(a.Y + rr), o1 = __ldg(a.W1 + rr), o2 = __ldg(a.W2 + rr);
    // ---- the previous iteration's scatter, while the loads are in flight
    if (SK && qprev >= 0) scatter(qprev, wprev);
    // ---- w_j at the own row and at the stencil columns (K2s's expression)
    double wo = c0 * oy;
    wo = fma(c2, o2, wo);
    wo = fma(c1, o1, wo);
    if (!live) wo = 0.0;
    double ys = 0.0;
#pragma unroll
    for (int k = 0; k < FMT; ++k) {
      double x = c0 * xy[k];
      x = fma(c2, x2[k], x);
      x = fma(c1, x1[k], x);
      ys = fma(v[k], x, ys);
    }
    if (live) {
      __stcs(a.Wout + row, wo);
      a.Ynew[row] = ys;
      acc[0] = fma(wo, wo, acc[0]);
      acc[1] = fma(wo, o1, acc[1]);
      acc[2] = fma(wo, o2, acc[2]);
      acc[3] = fma(ys, ys, acc[3]);
      acc[4] = fma(ys, wo, acc[4]);
      acc[5] = fma(ys, o1, acc[5]);
    }
    if (SK) {
      xbuf[stage * 64 + c * 32 + lane] = wo;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + p) : "memory");
      const double wpart = xbuf[stage * 64 + (1 - c) * 32 + lane];
      wprev[c] = wo;
      wprev[1 - c] = wpart;
      qprev = q;
      stage ^= 1;
    }
  }
  if (SK && qprev >= 0) scatter(qprev, wprev);
  // block partials (value-major)
  __shared__ double red[6][32];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double t = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = t;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int w = 0; w < 2 * PAIRS; ++w) t += red[threadIdx.x][w];
    a.partials[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (SK) {
    for (int r = warp; r < s; r += 2 * PAIRS) {
      double t = 0.0;
      for (int pp = 0; pp < PAIRS; ++pp) t += warp_sum(smem[(static_cast<int64_t>(pp) * s + r) * 32 + lane]);
      if (lane == 0) a.skp[static_cast<int64_t>(blockIdx.x) * s + r] = t;
    }
  }
}

// K1 as in spmv.cu MODE 1 (one x vector, window dot with W1), for calibration
template <int FMT>
__global__ void __launch_bounds__(256, 3) k_k1(Args a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double acc[3] = {0, 0, 0};
  int nx_off = 0;
  if (gw < a.nslices && lane < FMT) nx_off = __ldg(a.doff + gw * FMT + lane);
  for (int64_t sl = gw; sl < a.nslices; sl += nwarps) {
    const int cur_off = nx_off;
    if (sl + nwarps < a.nslices && lane < FMT) nx_off = __ldg(a.doff + (sl + nwarps) * FMT + lane);
    const int64_t row = sl * kSlice + lane;
    const bool live = row < a.nrows;
    const double e0 = live ? a.W1[row] : 0.0;
    const double e1 = live ? __ldcs(a.W2 + row) : 0.0;
    const double* vp = a.vals + sl * kSlice * FMT + lane;
    double v[FMT], xv[FMT];
#pragma unroll
    for (int k = 0; k < FMT; ++k) {
      const int o = __shfl_sync(0xffffffffu, cur_off, k);
      int64_t cidx = row + o;
      cidx = cidx < 0 ? 0 : (cidx >= a.ext_len ? a.ext_len - 1 : cidx);
      v[k] = __ldcs(vp + k * kSlice);
      xv[k] = __ldg(a.W1 + cidx);
    }
    double ys = 0.0;
#pragma unroll
    for (int k = 0; k < FMT; ++k) ys = fma(v[k], xv[k], ys);
    if (live) {
      a.Ynew[row] = ys;
      acc[0] = fma(ys, ys, acc[0]);
      acc[1] = fma(ys, e0, acc[1]);
      acc[2] = fma(ys, e1, acc[2]);
    }
  }
  __shared__ double red[3][8];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double t = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = t;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    a.partials[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_fill(double* p, int64_t n, uint64_t seed, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = scale * ((double)(mix64(seed + i) >> 11) * (1.0 / 9007199254740992.0) - 0.5);
}
__global__ void k_fill_off(int32_t* d, int64_t nslices) {
  const int off[7] = {-262144, -512, -1, 0, 1, 512, 262144};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslices * 7; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = off[i % 7];
}

template <class K>
float time_it(K launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  launch();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <int PAIRS, bool SK>
void run_fused(Args a, int nsm, double bytes, const char* name) {
  auto kern = k_fused<7, PAIRS, SK>;
  const size_t smem = sizeof(double) * (size_t(PAIRS) * a.s * 32 + PAIRS * 128);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 64 * PAIRS, smem));
  const int g = nsm * per;
  float ms = time_it([&] { kern<<<g, 64 * PAIRS, smem>>>(a); }, 5);
  CK(cudaGetLastError());
  printf("%-28s pairs=%d ctas/sm=%d  %.3f ms  %.0f GB/s\n", name, PAIRS, per, ms, bytes / ms * 1e-6);
}

int main(int argc, char** argv) {
  const int64_t L = argc > 1 ? atoll(argv[1]) : 512;
  const int64_t N = L * L * L, ns = N / 32;
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double *vals, *Y, *W1, *W2, *Wout, *Ynew, *part, *skp;
  int32_t* doff;
  CK(cudaMalloc(&vals, sizeof(double) * ns * 7 * 32));
  CK(cudaMalloc(&doff, sizeof(int32_t) * ns * 7));
  for (double** p : {&Y, &W1, &W2, &Wout, &Ynew}) CK(cudaMalloc(p, sizeof(double) * N));
  CK(cudaMalloc(&part, sizeof(double) * 6 * 4096));
  CK(cudaMalloc(&skp, sizeof(double) * 4096 * 128));
  k_fill<<<4096, 256>>>(vals, ns * 7 * 32, 1, 1.0);
  k_fill_off<<<4096, 256>>>(doff, ns);
  k_fill<<<4096, 256>>>(Y, N, 2, 1.0);
  k_fill<<<4096, 256>>>(W1, N, 3, 1.0);
  k_fill<<<4096, 256>>>(W2, N, 4, 1.0);
  CK(cudaDeviceSynchronize());
  Args a{vals, doff, N, ns, N, Y, W1, W2, Wout, Ynew, 0.7, -0.3, 0.1, part, skp, 0x1234567ull, 120};
  const double bA = 8.0 * ns * 7 * 32, bv = 8.0 * N;
  {
    const int per = 3, g = nsm * per;
    float ms = time_it([&] { k_k1<7><<<g, 256>>>(a); }, 5);
    CK(cudaGetLastError());
    printf("%-28s %.3f ms  %.0f GB/s\n", "K1 (x + 2 window)", ms, (bA + 4 * bv) / ms * 1e-6);
  }
  const double bF = bA + 5 * bv;
  run_fused<1, false>(a, nsm, bF, "fused, no sketch");
  run_fused<2, false>(a, nsm, bF, "fused, no sketch");
  run_fused<1, true>(a, nsm, bF, "fused + sparse sign");
  run_fused<2, true>(a, nsm, bF, "fused + sparse sign");
  run_fused<3, true>(a, nsm, bF, "fused + sparse sign");
  return 0;
}
