// PCIe copy bandwidth of pinned host memory: 1D vs 2D (row-strided) copies, both directions.
//   nvcc -O2 -o /tmp/copy_bw tools/copy_bw.cu && /tmp/copy_bw
#include <cuda_runtime.h>
#include <cstdio>

int main() {
  const size_t total = 38u << 20;  // ~ one 256-bit 1024^2 operand's SoA planes
  void *h, *d;
  cudaMallocHost(&h, 2 * total);
  cudaMalloc(&d, 2 * total);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* what, auto f) {
    for (int w = 0; w < 2; ++w) f();
    cudaEventRecord(a, s);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"copy\": \"%s\", \"GB_per_s\": %.1f}\n", what, 5.0 * total / (ms * 1e-3) / 1e9);
  };
  run("h2d 1d", [&] { cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s); });
  run("d2h 1d", [&] { cudaMemcpyAsync(h, d, total, cudaMemcpyDeviceToHost, s); });
  for (size_t wbytes : {512, 2048, 4096, 16384}) {
    const size_t rows = total / wbytes;
    char buf[64];
    snprintf(buf, sizeof buf, "h2d 2d rows of %zu B (pitch 2x)", wbytes);
    run(buf, [&] { cudaMemcpy2DAsync(d, wbytes, h, 2 * wbytes, wbytes, rows, cudaMemcpyHostToDevice, s); });
    snprintf(buf, sizeof buf, "d2h 2d rows of %zu B (pitch 2x)", wbytes);
    run(buf, [&] { cudaMemcpy2DAsync(h, 2 * wbytes, d, wbytes, wbytes, rows, cudaMemcpyDeviceToHost, s); });
  }
  // both directions at once (separate copy engines)
  cudaStream_t s2;
  cudaStreamCreate(&s2);
  cudaEventRecord(a, s);
  cudaStreamWaitEvent(s2, a, 0);
  for (int r = 0; r < 5; ++r) {
    cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((char*)h + total, (char*)d + total, total, cudaMemcpyDeviceToHost, s2);
  }
  cudaEventRecord(b, s2);
  cudaStreamWaitEvent(s, b, 0);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"copy\": \"h2d + d2h concurrent\", \"GB_per_s_each\": %.1f}\n", 5.0 * total / (ms * 1e-3) / 1e9);
  return 0;
}
