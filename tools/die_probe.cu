// Probe: which SMs share an L2 partition (die) on this B200?
//
// For each of L test lines (one 128-B line in each of L distinct 2 MB pages),
// every SM in turn (serialised by a ticket so only one SM probes at a time)
// times a chain of dependent L2-only loads (ld.global.cg bypasses L1) to that
// line.  An L2 hit in the near partition is faster than one that crosses the
// die-to-die link, so for each line the SMs split into two latency groups;
// the grouping (up to a flip) is the SM → die map, and the line's fast group
// tells its home die.  Output: lat[sm][line] in cycles (CSV on stdout).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/die_probe tools/die_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void probe(unsigned long long *buf, long long stride_elems, int n_lines, int chain, unsigned *ticket,
                      unsigned *order, long long *lat, int *sm_of_block) {
  if (threadIdx.x != 0) return;
  const unsigned sm = smid();
  sm_of_block[blockIdx.x] = sm;
  // wait for our turn (blocks probe one at a time)
  while (atomicAdd(ticket, 0) != blockIdx.x) __nanosleep(100);
  for (int l = 0; l < n_lines; ++l) {
    unsigned long long *p = buf + (long long)l * stride_elems;
    unsigned long long v = 0;
    // warm (also makes the line's value a self-pointer offset of 0)
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    long long t0 = clock64();
    for (int c = 0; c < chain; ++c) {
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p + v));  // v == 0: dependent chain
    }
    long long t1 = clock64();
    lat[(long long)blockIdx.x * n_lines + l] = (t1 - t0) / chain + (long long)(v & 1);
  }
  __threadfence();
  atomicAdd(ticket, 1u);
  (void)order;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n_lines = 64, chain = 256;
  const long long stride = (2ll << 20) / 8 + 16;  // 2 MB + 128 B apart (different pages and slices)
  unsigned long long *buf;
  cudaMalloc(&buf, (size_t)stride * 8 * n_lines + 4096);
  cudaMemset(buf, 0, (size_t)stride * 8 * n_lines + 4096);
  unsigned *ticket;
  cudaMalloc(&ticket, 8);
  cudaMemset(ticket, 0, 8);
  long long *lat;
  cudaMalloc(&lat, sizeof(long long) * sms * n_lines);
  int *sm_of;
  cudaMalloc(&sm_of, sizeof(int) * sms);
  // one block per SM: 1 block of 32 threads with enough smem that two cannot share an SM
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<sms, 32, 200 * 1024>>>(buf, stride, n_lines, chain, ticket, nullptr, lat, sm_of);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<long long> h(sms * n_lines);
  std::vector<int> s(sms);
  cudaMemcpy(h.data(), lat, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), sm_of, sizeof(int) * sms, cudaMemcpyDeviceToHost);
  printf("sm");
  for (int l = 0; l < n_lines; ++l) printf(",l%d", l);
  printf("\n");
  for (int b = 0; b < sms; ++b) {
    printf("%d", s[b]);
    for (int l = 0; l < n_lines; ++l) printf(",%lld", h[(size_t)b * n_lines + l]);
    printf("\n");
  }
  return 0;
}
