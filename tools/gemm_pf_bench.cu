// K8 harness (tools only): correctness of gemm_pf (csrc/gemm_pf.cu) against
// cuBLAS on the same bf16 operands, and CUDA-event timing of both over the
// Llama-3.1-8B projection shapes. Weights rotate over copies totalling
// >= 512 MB so every launch streams them from HBM as in a forward.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I paper_2410_01228_b200/csrc tools/gemm_pf_bench.cu paper_2410_01228_b200/csrc/gemm_pf.cu \
//        -lcublas -o tools/gemm_pf_bench
#include <cublas_v2.h>
#include <cuda.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace csk {
void gemm_pf(const CUtensorMap* xmap, const CUtensorMap* wmap, void* y, int M, const int32_t* m_dev, int N, int K,
             bool f32_out, int sms, cudaStream_t s, bool swiglu);
}

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

static bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void fill(__nv_bfloat16* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = __float2bfloat16(csk::hash_uniform(seed, 7, i));
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 20;
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cublasHandle_t h;
  cublasCreate(&h);
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cublasSetStream(h, s);
  void* ws;
  CK(cudaMalloc(&ws, 64 << 20));
  cublasSetWorkspace(h, ws, 64 << 20);
  struct Shape {
    const char* name;
    int N, K;
  };
  const Shape shapes[] = {{"qkv", 6144, 4096}, {"o_proj", 4096, 4096}, {"gate_up", 28672, 4096}, {"down", 4096, 14336}};
  const int Ms[] = {256, 512, 1000, 2048, 3000, 4096, 8192};
  int32_t* d_m;
  CK(cudaMalloc(&d_m, 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::printf("shape M N K | max|diff| max|ref| | K8 ms TFLOP/s | cuBLAS ms TFLOP/s | K8/cuBLAS\n");
  int bad = 0;
  for (const Shape& sh : shapes) {
    const size_t nw = static_cast<size_t>(sh.N) * sh.K;
    const int copies = static_cast<int>(std::max<size_t>(1, ((512ull << 20) + nw * 2 - 1) / (nw * 2)));
    __nv_bfloat16 *w, *x, *y1, *y2;
    const int Mmax = 8192;
    CK(cudaMalloc(&w, nw * 2 * copies));
    CK(cudaMalloc(&x, static_cast<size_t>(Mmax) * sh.K * 2));
    CK(cudaMalloc(&y1, static_cast<size_t>(Mmax) * sh.N * 2));
    CK(cudaMalloc(&y2, static_cast<size_t>(Mmax) * sh.N * 2));
    fill<<<1024, 256, 0, s>>>(w, nw * copies, 1);
    fill<<<1024, 256, 0, s>>>(x, static_cast<size_t>(Mmax) * sh.K, 2);
    std::vector<CUtensorMap> wm(copies);
    for (int c = 0; c < copies; ++c)
      if (!make_map(&wm[c], w + nw * c, sh.N, sh.K, 128)) std::printf("map fail\n");
    CUtensorMap xm;
    make_map(&xm, x, Mmax, sh.K, 128);
    for (int M : Ms) {
      // device M smaller than the host bound for one case: tiles past it must not be written
      CK(cudaMemsetAsync(y1, 0, static_cast<size_t>(M) * sh.N * 2, s));
      CK(cudaMemcpyAsync(d_m, &M, 4, cudaMemcpyHostToDevice, s));
      csk::gemm_pf(&xm, &wm[0], y1, Mmax, d_m, sh.N, sh.K, false, sms, s, false);
      const float alpha = 1.f, beta = 0.f;
      cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, sh.N, M, sh.K, &alpha, w, CUDA_R_16BF, sh.K, x, CUDA_R_16BF, sh.K,
                   &beta, y2, CUDA_R_16BF, sh.N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
      CK(cudaStreamSynchronize(s));
      CK(cudaGetLastError());
      std::vector<__nv_bfloat16> a(static_cast<size_t>(M) * sh.N), b(a.size());
      CK(cudaMemcpy(a.data(), y1, a.size() * 2, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b.data(), y2, b.size() * 2, cudaMemcpyDeviceToHost));
      double md = 0, mr = 0;
      for (size_t i = 0; i < a.size(); ++i) {
        const double u = __bfloat162float(a[i]), v = __bfloat162float(b[i]);
        md = std::max(md, std::fabs(u - v));
        mr = std::max(mr, std::fabs(v));
      }
      if (!(md <= 2e-2 * mr + 1e-3)) ++bad;
      auto timeit = [&](bool k8) {
        for (int r = 0; r < 3 + reps; ++r) {
          if (r == 3) CK(cudaEventRecord(e0, s));
          if (k8) {
            csk::gemm_pf(&xm, &wm[r % copies], y1, M, nullptr, sh.N, sh.K, false, sms, s, false);
          } else {
            cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, sh.N, M, sh.K, &alpha, w + nw * (r % copies), CUDA_R_16BF,
                         sh.K, x, CUDA_R_16BF, sh.K, &beta, y2, CUDA_R_16BF, sh.N, CUBLAS_COMPUTE_32F,
                         CUBLAS_GEMM_DEFAULT);
          }
        }
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms / reps;
      };
      const double t8 = timeit(true), tb = timeit(false);
      const double fl = 2.0 * M * sh.N * sh.K;
      std::printf("%-8s %5d %6d %6d | %.3g %.3g | %.4f %7.1f | %.4f %7.1f | %.3f\n", sh.name, M, sh.N, sh.K, md, mr,
                  t8, fl / t8 / 1e9, tb, fl / tb / 1e9, tb / t8);
      std::fflush(stdout);
    }
    cudaFree(w);
    cudaFree(x);
    cudaFree(y1);
    cudaFree(y2);
  }
  std::printf("RESULT %s\n", bad ? "MISMATCH" : "ok");
  return bad ? 1 : 0;
}
