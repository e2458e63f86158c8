// Which SASS operations issue on which pipe on this GPU (ncu pipe metrics per kernel).
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double ctab[256];
__global__ void k_dsetp(const double* x, int* out, double t, int it) {
  double v[8]; int c = 0;
  for (int i = 0; i < 8; ++i) v[i] = x[threadIdx.x + i];
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { c += fabs(v[i]) > t; v[i] = -v[i]; }
  }
  out[threadIdx.x] = c;
}
__global__ void k_popc(const unsigned* x, int* out, int it) {
  unsigned v[8]; int c = 0;
  for (int i = 0; i < 8; ++i) v[i] = x[threadIdx.x + i];
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { c += __popc(v[i]); v[i] = v[i] * 3u + 1u; }
  }
  out[threadIdx.x] = c;
}
__global__ void k_ldc(int* out, int it) {
  double s = 0.0; int j = threadIdx.x & 255;
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { s += ctab[(j + i * 7 + k) & 255]; }
  }
  out[threadIdx.x] = (int)s;
}
__global__ void k_zero64(double* out, const double* x, int it) {
  double acc = 0.0;
  for (int k = 0; k < it; ++k) {
    double2 z[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] = (k + i) & 1 ? make_double2(0.0, 0.0) : make_double2(x[i], x[i + 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc += z[i].x * z[i].y;
  }
  out[threadIdx.x] = acc;
}
__global__ void k_dadd(const double* x, double* out, int it) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = x[threadIdx.x + i];
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __dadd_rn(v[i], 1.0);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  out[threadIdx.x] = s;
}
__global__ void k_shfl(int* out, int it) {
  int v[8]; for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_xor_sync(0xffffffffu, v[i], 1 + i) + 1;
  }
  int s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  out[threadIdx.x] = s;
}
__global__ void k_ballot(const double* x, int* out, double t, int it) {
  double v[8]; int c = 0;
  for (int i = 0; i < 8; ++i) v[i] = x[threadIdx.x + i];
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { c += __ballot_sync(0xffffffffu, v[i] > t) & 3; v[i] += 1.0; }
  }
  out[threadIdx.x] = c;
}
int main() {
  double* x; int* o; double* od; unsigned* u;
  cudaMalloc(&x, 4096 * 8); cudaMalloc(&o, 4096 * 4); cudaMalloc(&od, 4096 * 8); cudaMalloc(&u, 4096 * 4);
  cudaMemset(x, 0, 4096 * 8); cudaMemset(u, 0, 4096 * 4);
  const int G = 148 * 4, B = 512, IT = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto f, double ops_per_thread_iter) {
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_ops = (double)G * B / 32 * IT * ops_per_thread_iter;
    printf("%-8s %8.3f ms  %.3f warp-ops/clk/SM (at 1.965 GHz)\n", name, ms, warp_ops / (ms * 1e-3 * 1.965e9) / 148);
  };
  run("dsetp", [&] { k_dsetp<<<G, B>>>(x, o, 0.5, IT); }, 8);
  run("popc", [&] { k_popc<<<G, B>>>(u, o, IT); }, 8);
  run("ldc", [&] { k_ldc<<<G, B>>>(o, IT); }, 8);
  run("zero64", [&] { k_zero64<<<G, B>>>(od, x, IT); }, 4);
  run("dadd", [&] { k_dadd<<<G, B>>>(x, od, IT); }, 8);
  run("shfl", [&] { k_shfl<<<G, B>>>(o, IT); }, 8);
  run("ballot", [&] { k_ballot<<<G, B>>>(x, o, 0.5, IT); }, 8);
  return 0;
}
