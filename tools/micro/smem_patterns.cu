// Shared-memory access-pattern microbenchmark (ncu: L1 wavefronts shared per instruction).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int T = 8192;
__global__ void k_lds_u8(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint8_t buf[T];
  for (int i = threadIdx.x; i < T; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  uint32_t acc = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += buf[(wid * 16 + e) * 32 + lane] ^ it;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds_u32(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint32_t buf[T / 4];
  for (int i = threadIdx.x; i < T / 4; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  uint32_t acc = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc += buf[(wid * 4 + e) * 32 + lane] ^ it;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_sts_u8_lin(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint8_t buf[T];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) buf[(wid * 16 + e) * 32 + ((lane + it) & 31)] = (uint8_t)(lane + e);
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = buf[threadIdx.x * 3 % T];
}
// two streams (zeros / ones) of consecutive bytes in distant regions
__global__ void k_sts_u8_split(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint8_t buf[T];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t m = 0x5a3c96e1u;
  const unsigned lt = (1u << lane) - 1u;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t mm = m ^ (e * 0x9e3779b9u) ^ it;
      const int b = (mm >> lane) & 1;
      const int r1 = __popc(mm & lt);
      const int base = (wid * 16 + e) * 16;
      const int dst = b ? (4096 + base + r1 + 7 * it) & (T - 1) : (base + lane - r1);
      buf[dst] = (uint8_t)(lane + e);
    }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = buf[threadIdx.x * 3 % T];
}
__global__ void k_sts_u32(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint32_t buf[T];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) buf[((wid * 16 + e) * 32 + ((lane + it) & 31)) & (T - 1)] = lane + e;
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = buf[threadIdx.x * 3 % T];
}
__global__ void k_shfl(const uint8_t* in, uint32_t* out, int iters) {
  uint32_t acc = threadIdx.x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += __shfl_sync(0xffffffffu, acc, (threadIdx.x + e) & 31);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_redux(const uint8_t* in, uint32_t* out, int iters) {
  uint32_t acc = threadIdx.x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += __reduce_or_sync(0xffffffffu, acc << (e & 7));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_vote(const uint8_t* in, uint32_t* out, int iters) {
  uint32_t acc = threadIdx.x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += __ballot_sync(0xffffffffu, (acc >> e) & 1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_match(const uint8_t* in, uint32_t* out, int iters) {
  uint32_t acc = threadIdx.x;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += __match_any_sync(0xffffffffu, (acc >> e) & 15);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_atoms(const uint8_t* in, uint32_t* out, int iters) {
  __shared__ uint32_t c[32][16];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&c[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) atomicAdd(&c[(e + it) & 31][(lane * 7 + e) & 15], 1u);
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[threadIdx.x & 31][threadIdx.x & 15];
}
__global__ void k_popc(const uint8_t* in, uint32_t* out, int iters) {
  uint32_t acc = threadIdx.x * 0x9e3779b9u;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int e = 0; e < 16; ++e) acc += __popc(acc ^ (e * 0x01010101u));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint8_t* in; uint32_t* out;
  cudaMalloc(&in, T); cudaMalloc(&out, 148 * 4 * 512 * 4);
  cudaMemset(in, 1, T);
  const int iters = 256;
  dim3 g(148 * 4), b(512);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(const uint8_t*, uint32_t*, int), int ops_per_iter) {
    k<<<g, b>>>(in, out, iters);
    cudaEventRecord(e0);
    k<<<g, b>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_ops = (double)g.x * (b.x / 32) * iters * ops_per_iter;
    double cyc = ms * 1e-3 * 1.965e9 * 148;
    printf("%-16s %8.3f ms  %6.2f SM-cycles per warp-op\n", name, ms, cyc / warp_ops);
  };
  run("lds_u8", k_lds_u8, 16);
  run("lds_u32", k_lds_u32, 4);
  run("sts_u8_lin", k_sts_u8_lin, 16);
  run("sts_u8_split", k_sts_u8_split, 16);
  run("sts_u32", k_sts_u32, 16);
  run("shfl", k_shfl, 16);
  run("redux_or", k_redux, 16);
  run("vote", k_vote, 16);
  run("match_any", k_match, 16);
  run("atoms", k_atoms, 16);
  run("popc", k_popc, 16);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
