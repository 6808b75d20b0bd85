// Probe: does any cuBLASLt algorithm beat the default heuristic choice for the
// encoder's bf16 GEMMs (y = x W^T + b, bias epilogue) at the bench shape?
// Build: nvcc -O2 -o gemm_algo_probe gemm_algo_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include <algorithm>

__global__ void fill(__nv_bfloat16* p, long n, unsigned seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = __float2bfloat16(((h & 0xffff) / 32768.f - 1.f));  // U(-1, 1): realistic tensor-core power
  }
}

#define CK(x) do { auto e = (x); if (e != 0) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); return 1; } } while (0)

int main() {
  const long M = 64L * 4099;  // tokens
  struct Shape { const char* name; long N, K; } shapes[] = {{"qkv", 2304, 768}, {"wo", 768, 768}, {"w1", 3072, 768}, {"w2", 768, 3072}};
  cublasLtHandle_t lt; CK(cublasLtCreate(&lt));
  size_t wsz = 64 << 20; void* ws; cudaMalloc(&ws, wsz);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& sh : shapes) {
    const long N = sh.N, K = sh.K;
    __nv_bfloat16 *A, *W, *D; float* bias_f; __nv_bfloat16* bias;
    cudaMalloc(&A, M * K * 2); cudaMalloc(&W, N * K * 2); cudaMalloc(&D, M * N * 2); cudaMalloc(&bias, N * 2);
    fill<<<1184, 256>>>(A, M * K, 1); fill<<<1184, 256>>>(W, N * K, 2); cudaMemset(bias, 0, N * 2);
    (void)bias_f;
    // column-major view: D^T[N,M] = W[N,K] (as op T of [K,N] col-major) * A^T[K,M]
    cublasLtMatmulDesc_t op; CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
    cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_BIAS;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias)));
    cudaDataType_t bt = CUDA_R_16BF;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)));
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K));   // W stored [N][K] row-major = [K,N] col-major
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, K));   // A [M][K] row-major = [K,M] col-major
    CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, N, M, N));   // D [M][N] row-major = [N,M] col-major
    cublasLtMatmulPreference_t pref; CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz)));
    cublasLtMatmulHeuristicResult_t res[32]; int n = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 32, res, &n));
    float alpha = 1.f, beta = 0.f;
    double flops = 2.0 * M * N * K;
    printf("%s M=%ld N=%ld K=%ld: %d algos\n", sh.name, M, N, K, n);
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      for (int r = 0; r < 3; ++r) cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, D, lc, D, lc, &res[i].algo, ws, wsz, 0);
      cudaEventRecord(e0);
      const int it = 10;
      for (int r = 0; r < it; ++r) cublasLtMatmul(lt, op, &alpha, W, la, A, lb, &beta, D, lc, D, lc, &res[i].algo, ws, wsz, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= it;
      int tile = 0, stages = 0, cga = 0; size_t sz;
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages, sizeof(stages), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID, &cga, sizeof(cga), &sz);
      printf("  algo %2d: %.3f ms  %.0f TFLOP/s  tile=%d stages=%d cluster=%d ws=%zu\n", i, ms, flops / ms / 1e9, tile, stages, cga, res[i].workspaceSize);
    }
    cudaFree(A); cudaFree(W); cudaFree(D); cudaFree(bias);
  }
  return 0;
}
