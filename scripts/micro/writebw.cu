// Write-bandwidth microbenchmark: which store structure reaches HBM peak?
//   A: grid-stride STG.128            B: grid-stride STG.256
//   C: per-warp 2 KB smem stage + cp.async.bulk store (our fill's structure)
//   D: same as C with 8 KB stages     E: C with evict_first hint
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void kA(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, 1, 2, 3);
}
__global__ void kB(float* p, size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    float* q = p + 8 * i; float a = (float)i;
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(q), "f"(a) : "memory");
  }
}
template <int STAGE, bool HINT>
__global__ void kC(uint8_t* p, size_t nchunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* buf = sm + w * 2 * STAGE;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int k = 0;
  size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  size_t tw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = gw; c < nchunks; c += tw, ++k) {
    uint8_t* b = buf + (k & 1) * STAGE;
    if (k >= 2) { if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); __syncwarp(); }
    for (int o = lane * 16; o < STAGE; o += 512) *reinterpret_cast<uint4*>(b + o) = make_uint4(c, o, 1, 2);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(b);
      if (HINT) asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" :: "l"(p + c * STAGE), "r"(sa), "r"(STAGE), "l"(pol) : "memory");
      else asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(p + c * STAGE), "r"(sa), "r"(STAGE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const size_t bytes = 470ull << 20;
  uint8_t* p; cudaMalloc(&p, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int i = 0; i < 10; ++i) { cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    printf("%-40s %8.1f GB/s  (%.1f us)  %s\n", name, bytes / (best * 1e-3) / 1e9, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  run("A STG.128 grid-stride 148x8x256", [&]{ kA<<<sms * 8, 256>>>((uint4*)p, bytes / 16); });
  run("B STG.256 grid-stride 148x8x256", [&]{ kB<<<sms * 8, 256>>>((float*)p, bytes / 32); });
  run("memset", [&]{ cudaMemsetAsync(p, 0, bytes); });
  for (int occ : {2, 4, 6}) {
    char nm[64];
    cudaFuncSetAttribute(kC<2048, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2 * 2048);
    snprintf(nm, 64, "C bulk 2KB stages, %d CTAx4w/SM", occ);
    run(nm, [&]{ kC<2048, false><<<sms * occ, 128, 4 * 2 * 2048>>>(p, bytes / 2048); });
    cudaFuncSetAttribute(kC<8192, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2 * 8192);
    snprintf(nm, 64, "D bulk 8KB stages, %d CTAx4w/SM", occ);
    run(nm, [&]{ kC<8192, false><<<sms * occ, 128, 4 * 2 * 8192>>>(p, bytes / 8192); });
    cudaFuncSetAttribute(kC<2048, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2 * 2048);
    snprintf(nm, 64, "E bulk 2KB evict_first, %d CTAx4w/SM", occ);
    run(nm, [&]{ kC<2048, true><<<sms * occ, 128, 4 * 2 * 2048>>>(p, bytes / 2048); });
  }
  return 0;
}
