// HBM streaming probe: how many SMs (and how many bytes in flight per SM) does a TMA weight stream need to reach
// the HBM roofline? Streams a [28672, 4096] bf16 matrix (235 MB, > L2) once per launch with G CTAs, each a single
// producer thread issuing 2-D tensor boxes (R rows x 64 bf16, 128 B swizzle: the GEMM's B operand box) or 1-D bulk
// copies into an S-stage ring, and a consumer thread releasing the stages (no math).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/probe/stream_bw \
//        tools/probe/stream_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2505_07203_b200/csrc/sm100.cuh"
using namespace po;

constexpr int NROWS = 28672, KCOLS = 4096;

template <bool TWO_D>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                               int rows_per_box, int stages, long long total_boxes) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int box_bytes = rows_per_box * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * box_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int kbs = KCOLS / 64;
  // contiguous range of boxes per CTA (box b: row block b / kbs, k block b % kbs)
  const long long lo = total_boxes * blockIdx.x / gridDim.x, hi = total_boxes * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0;
    for (long long b = lo; b < hi; ++b) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], box_bytes);
      if (TWO_D) {
        tma_load_2d(smem + s * box_bytes, &map, &full[s], (int)(b % kbs) * 64, (int)(b / kbs) * rows_per_box);
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(smem + s * box_bytes)), "l"(src + b * box_bytes), "r"(box_bytes),
                     "r"(smem_u32(&full[s])) : "memory");
      }
      if (++s == stages) { s = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0;
    for (long long b = lo; b < hi; ++b) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == stages) { s = 0; ph ^= 1; }
    }
  }
}

__global__ void read_flush(const int4* p, long long n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int4 v = p[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffff) *sink = 1;
}

int main() {
  int* sink; cudaMalloc(&sink, 4);
  void* w; cudaMalloc(&w, (size_t)NROWS * KCOLS * 2);
  cudaMemset(w, 1, (size_t)NROWS * KCOLS * 2);
  void* flush; cudaMalloc(&flush, 512ull << 20);
  cudaMemset(flush, 0, 512ull << 20);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = (double)NROWS * KCOLS * 2;
  for (int two_d = 1; two_d >= 0; --two_d)
    for (int rows : {128, 256})
      for (int stages : {2, 4, 6}) {
        const int box = rows * 128;
        const int smem = stages * box + 1024 + 256;
        if (smem > 227 * 1024) continue;
        CUtensorMap map;
        cuuint64_t dims[2] = {KCOLS, NROWS}; cuuint64_t str[1] = {KCOLS * 2};
        cuuint32_t bx[2] = {64, (cuuint32_t)rows}; cuuint32_t es[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        auto kern = two_d ? probe<true> : probe<false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const long long total = (long long)(NROWS / rows) * (KCOLS / 64);
        printf("%s rows=%d stages=%d (%d KB in flight/SM):", two_d ? "2D" : "1D", rows, stages, stages * box / 1024);
        for (int g : {8, 16, 32, 48, 64, 96, 128, nsm}) {
          std::vector<float> ts;
          for (int r = 0; r < 5; ++r) {
            read_flush<<<nsm * 4, 512>>>((const int4*)flush, (512ll << 20) / 16, sink);  // a read: no dirty lines
            cudaEventRecord(e0);
            kern<<<g, 64, smem>>>(map, (const uint8_t*)w, rows, stages, total);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
          }
          std::sort(ts.begin(), ts.end());
          printf("  %d:%.0f", g, bytes / (ts[2] * 1e-3) / 1e9);
        }
        printf("  GB/s\n");
        fflush(stdout);
      }
  cudaError_t err = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(err));
}
