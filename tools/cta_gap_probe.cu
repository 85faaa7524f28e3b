// CTA turnover probe: how long does an SM take to start the next CTA of a grid after one
// retires?  Non-persistent kernels with 2 CTAs per SM (the forward's shape: 224 threads,
// ~97 KB of dynamic smem) whose CTAs spin for a fixed time; variants add TMEM alloc/dealloc
// and a TMA-free global store tail.  Prints the median retire -> next-entry gap per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cta_gap_probe tools/cta_gap_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(224, 2) k_probe(unsigned long long* out, int spin_ns, float* sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t holder;
  const uint64_t t_entry = gtime();
  if (MODE >= 1) {
    if (threadIdx.x / 32 == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&holder)),
                   "r"(256)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  __syncthreads();
  const uint64_t t0 = gtime();
  while (gtime() - t0 < (uint64_t)spin_ns) {
  }
  if (MODE >= 2) sink[blockIdx.x * 224 + threadIdx.x] = (float)smem[threadIdx.x];
  __syncthreads();
  const uint64_t t1 = gtime();
  if (MODE >= 1) {
    if (threadIdx.x / 32 == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(holder), "r"(256) : "memory");
  }
  if (threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    out[blockIdx.x * 4 + 0] = t_entry;
    out[blockIdx.x * 4 + 1] = t1;
    out[blockIdx.x * 4 + 2] = sm;
  }
}

template <int MODE>
void run(const char* name, int grid, int smem, int spin_ns, unsigned long long* d_out, float* d_sink) {
  cudaFuncSetAttribute(k_probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) k_probe<MODE><<<grid, 224, smem>>>(d_out, spin_ns, d_sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  std::vector<unsigned long long> h(grid * 4);
  cudaMemcpy(h.data(), d_out, grid * 4 * 8, cudaMemcpyDeviceToHost);
  std::vector<double> gaps;
  int nsm = 0;
  for (auto i = 0; i < grid; ++i) nsm = std::max<int>(nsm, (int)h[i * 4 + 2] + 1);
  for (int s = 0; s < nsm; ++s) {
    std::vector<unsigned long long> st, en;
    for (int i = 0; i < grid; ++i)
      if ((int)h[i * 4 + 2] == s) {
        st.push_back(h[i * 4]);
        en.push_back(h[i * 4 + 1]);
      }
    std::sort(st.begin(), st.end());
    std::sort(en.begin(), en.end());
    for (size_t k = 2; k < st.size(); ++k) gaps.push_back((double)(st[k] - en[k - 2]) / 1e3);
  }
  std::sort(gaps.begin(), gaps.end());
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int i = 0; i < grid; ++i) {
    t0 = std::min(t0, h[i * 4]);
    t1 = std::max(t1, h[i * 4 + 1]);
  }
  printf("%-34s grid %5d smem %6d spin %6d ns: span %8.1f us, retire->entry gap median %.2f us p90 %.2f us\n", name,
         grid, smem, spin_ns, (t1 - t0) / 1e3, gaps.empty() ? 0 : gaps[gaps.size() / 2],
         gaps.empty() ? 0 : gaps[gaps.size() * 9 / 10]);
}

// Divergent-arrival check: lane 0 of warp 2 spins 5 us longer than everyone else, sets a
// shared flag and stamps the timer, then reaches __syncthreads; thread 0 reads the flag and
// stamps after it.  Done once as the kernel's first barrier (phase 0) and once after another
// barrier (phase 1).  A working barrier never lets thread 0 miss the flag.
__global__ void k_bar(unsigned long long* out) {
  __shared__ volatile int flag[2];
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) flag[0] = flag[1] = 0;  // (no barrier yet: the spinner writes 5 us later)
  for (int ph = 0; ph < 2; ++ph) {
    if (warp == 2 && (threadIdx.x & 31) == 0) {
      const uint64_t t0 = gtime();
      while (gtime() - t0 < 5000) {
      }
      flag[ph] = 1;
      out[(blockIdx.x * 2 + ph) * 4 + 0] = gtime();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      out[(blockIdx.x * 2 + ph) * 4 + 1] = gtime();
      out[(blockIdx.x * 2 + ph) * 4 + 2] = flag[ph];
    }
  }
}

int main() {
  {
    unsigned long long* d;
    cudaMalloc(&d, 1024 * 8 * 8);
    k_bar<<<1024, 224>>>(d);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(1024 * 8);
    cudaMemcpy(h.data(), d, 1024 * 8 * 8, cudaMemcpyDeviceToHost);
    for (int ph = 0; ph < 2; ++ph) {
      int early = 0, noflag = 0;
      for (int i = 0; i < 1024; ++i) {
        const unsigned long long* r = &h[(i * 2 + ph) * 4];
        early += r[1] < r[0];
        noflag += r[2] != 1;
      }
      printf("barrier check phase %d: thread 0 stamped before the late lane in %d of 1024 CTAs, missed its flag in %d\n",
             ph, early, noflag);
    }
  }
  const int grid = 3072;
  unsigned long long* d_out;
  float* d_sink;
  cudaMalloc(&d_out, grid * 4 * 8);
  cudaMalloc(&d_sink, grid * 224 * 4);
  for (int smem : {97 * 1024}) {
    for (int spin : {2000, 20000}) {
      run<0>("plain", grid, smem, spin, d_out, d_sink);
      run<1>("tmem alloc/dealloc", grid, smem, spin, d_out, d_sink);
      run<2>("tmem + global store tail", grid, smem, spin, d_out, d_sink);
    }
  }
  return 0;
}
