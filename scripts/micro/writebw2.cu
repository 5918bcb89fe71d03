// Store-pattern study: what reaches memset's write bandwidth?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// F: each warp writes a contiguous CH-byte chunk per iteration (unrolled STG.128)
template <int CH, int MODE>
__global__ void kF(uint8_t* p, size_t nch) {
  const int lane = threadIdx.x & 31;
  size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  size_t tw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = gw; c < nch; c += tw) {
    uint4* q = reinterpret_cast<uint4*>(p + c * CH);
#pragma unroll
    for (int k = 0; k < CH / 512; ++k) {
      uint4 v = make_uint4(c, k, lane, 7);
      if (MODE == 0) q[k * 32 + lane] = v;
      else if (MODE == 1) __stcs(q + k * 32 + lane, v);
      else asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(q + k * 32 + lane), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
  }
}
// H: each block owns a contiguous region, writes it front to back
__global__ void kH(uint4* p, size_t n_per_block) {
  uint4* q = p + blockIdx.x * n_per_block;
  for (size_t i = threadIdx.x; i < n_per_block; i += blockDim.x) q[i] = make_uint4(i, 1, 2, 3);
}
int main() {
  const size_t bytes = 470ull << 20;
  uint8_t* p; cudaMalloc(&p, bytes + (64 << 20));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int i = 0; i < 10; ++i) { cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    printf("%-44s %8.1f GB/s  (%.1f us)  %s\n", name, bytes / (best * 1e-3) / 1e9, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  run("memset", [&]{ cudaMemsetAsync(p, 0, bytes); });
  run("memset 0x5a", [&]{ cudaMemsetAsync(p, 0x5a, bytes); });
  for (int g : {1, 2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "F 4KB/warp-iter default, %d blk/SM", g);
    run(nm, [&]{ kF<4096, 0><<<sms * g, 256>>>(p, bytes / 4096); });
    snprintf(nm, 64, "F 4KB/warp-iter .cs, %d blk/SM", g);
    run(nm, [&]{ kF<4096, 1><<<sms * g, 256>>>(p, bytes / 4096); });
    snprintf(nm, 64, "F 16KB/warp-iter default, %d blk/SM", g);
    run(nm, [&]{ kF<16384, 0><<<sms * g, 256>>>(p, bytes / 16384); });
  }
  for (int nb : {148, 592, 2368, 9472}) {
    char nm[64]; snprintf(nm, 64, "H block-contiguous, %d blocks", nb);
    size_t per = bytes / 16 / nb;
    run(nm, [&]{ kH<<<nb, 256>>>((uint4*)p, per); });
  }
  return 0;
}
