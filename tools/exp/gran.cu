// DRAM fetch-granularity probe (development): each thread copies a 96-byte
// span (6 x 16 B cp.async-sized loads) of "its grid" at stride S starting at
// a pseudo-random in-grid offset, like step_main's view window.  Compare ncu
// dram__bytes_read.sum for S = 169 (packed) and S = 192 / 256 (64-B aligned).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void probe(const uint8_t* g, int64_t n, int S, int span, uint32_t* out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint32_t h = (uint32_t)e * 2654435761u;
  int off = (int)(h % (uint32_t)(169 - span + 1));
  uintptr_t a = reinterpret_cast<uintptr_t>(g + e * S + off) & ~uintptr_t(15);
  uint32_t acc = 0;
  for (int k = 0; k < (span + 31) / 16; ++k) {
    uint4 v = __ldcg(reinterpret_cast<const uint4*>(a) + k);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  out[e] = acc;
}
int main() {
  const int64_t n = 1 << 20;
  uint8_t* g; uint32_t* out;
  cudaMalloc(&g, n * 256 + 256);
  cudaMalloc(&out, n * 4);
  cudaMemset(g, 1, n * 256 + 256);
  for (int S : {169, 176, 192, 256}) {
    for (int rep = 0; rep < 3; ++rep) probe<<<(n + 255) / 256, 256>>>(g, n, S, 70, out);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<(n + 255) / 256, 256>>>(g, n, S, 70, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("S=%d: %.1f us\n", S, ms * 1e3);
  }
  return 0;
}
