// L2 topology probe (experiment, not product): (1) DRAM bytes when many SMs read one buffer
// (unified vs per-die L2 caching, capacity), (2) per-SM L2-hit latency to single lines (die map).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_die_probe l2_die_probe.cu
// ./l2_die_probe read SIZE_MB PASSES MODE   (MODE 0 all SMs, 1 smid < 74, 2 even smid, 3 die-0 list)
// ./l2_die_probe lat NLINES
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 v; asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v;
}

__global__ void rd(const uint4* p, size_t n16, int passes, int mode, unsigned* sink, const int* die) {
  const unsigned s = smid();
  if (mode == 1 && s >= 74) return;
  if (mode == 2 && (s & 1)) return;
  if (mode == 3 && die[s] != 0) return;
  if (mode == 4) {                       // die d reads half d of the buffer
    n16 /= 2; p += die[s] * n16;
  }
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t start = (n16 / gridDim.x) * blockIdx.x;
  for (int ps = 0; ps < passes; ++ps)
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
      size_t j = start + i; if (j >= n16) j -= n16;
      uint4 v = ld_cg(p + j);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = 1;
}

// per-SM latency of dependent loads to line `l` (each line holds its own address)
__global__ void lat(unsigned long long* lines, int nlines, int iters, unsigned* out_smid, float* out_cyc) {
  if (threadIdx.x != 0) return;
  for (int l = 0; l < nlines; ++l) {
    unsigned long long* p = lines + l * 32;      // 256-byte stride
    unsigned long long a = (unsigned long long)p;
    for (int w = 0; w < 4; ++w) asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) asm volatile("ld.global.cg.u64 %0, [%0];" : "+l"(a));
    long long t1 = clock64();
    out_cyc[blockIdx.x * nlines + l] = (float)(t1 - t0) / iters + (a == 1 ? 1.f : 0.f);
  }
  out_smid[blockIdx.x] = smid();
}

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink; cudaMalloc(&sink, 4);
  if (!strcmp(argv[1], "read")) {
    size_t bytes = (size_t)atoi(argv[2]) << 20; int passes = atoi(argv[3]), mode = atoi(argv[4]);
    void* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
    // die map: per-SM latency to one line, split at the midpoint
    unsigned long long* line; cudaMalloc(&line, 256);
    unsigned long long hl = (unsigned long long)line; cudaMemcpy(line, &hl, 8, cudaMemcpyHostToDevice);
    unsigned* os; float* oc; cudaMalloc(&os, sms * 4); cudaMalloc(&oc, sms * 4);
    lat<<<sms, 32>>>(line, 1, 256, os, oc); cudaDeviceSynchronize();
    std::vector<unsigned> hs(sms); std::vector<float> hc(sms);
    cudaMemcpy(hs.data(), os, sms * 4, cudaMemcpyDeviceToHost); cudaMemcpy(hc.data(), oc, sms * 4, cudaMemcpyDeviceToHost);
    float mn = 1e9, mx = 0; for (float c : hc) { mn = c < mn ? c : mn; mx = c > mx ? c : mx; }
    std::vector<int> hd(256, 0); int n0 = 0;
    for (int b = 0; b < sms; ++b) { hd[hs[b]] = hc[b] > (mn + mx) / 2; n0 += hd[hs[b]] == 0; }
    printf("die 0: %d SMs, die 1: %d SMs (lat %.0f / %.0f)\n", n0, sms - n0, mn, mx);
    int* dd; cudaMalloc(&dd, 256 * 4); cudaMemcpy(dd, hd.data(), 256 * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    rd<<<sms, 1024, 200 * 1024>>>((const uint4*)p, bytes / 16, passes, mode, sink, dd);   // one CTA per SM
    cudaError_t e = cudaDeviceSynchronize(); printf("read %zu MB passes %d mode %d: %s\n", bytes >> 20, passes, mode, cudaGetErrorString(e));
  } else {
    int nl = atoi(argv[2]);
    unsigned long long* lines; cudaMalloc(&lines, (size_t)nl * 256);
    std::vector<unsigned long long> h(nl * 32);
    for (int l = 0; l < nl; ++l) h[l * 32] = (unsigned long long)(lines + l * 32);
    cudaMemcpy(lines, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    unsigned* os; float* oc; cudaMalloc(&os, sms * 4); cudaMalloc(&oc, sms * nl * 4);
    cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    lat<<<sms, 32, 200 * 1024>>>(lines, nl, 256, os, oc);
    cudaDeviceSynchronize();
    std::vector<unsigned> hs(sms); std::vector<float> hc(sms * nl);
    cudaMemcpy(hs.data(), os, sms * 4, cudaMemcpyDeviceToHost); cudaMemcpy(hc.data(), oc, sms * nl * 4, cudaMemcpyDeviceToHost);
    for (int b = 0; b < sms; ++b) {
      printf("smid %3u:", hs[b]);
      for (int l = 0; l < nl; ++l) printf(" %5.0f", hc[b * nl + l]);
      printf("\n");
    }
  }
  return 0;
}
