// Standalone TMA sanity test (debug helper): modes select where the tensor map
// lives and which coordinates are used.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
struct alignas(64) P { CUtensorMap m; const CUtensorMap* gm; float* out; int n; int x0, y0; int use_global; };
__global__ void k(const __grid_constant__ P p) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned s = (unsigned)__cvta_generic_to_shared(sm);
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const CUtensorMap* mp = p.use_global ? p.gm : &p.m;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(p.n*4) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      :: "r"(s), "l"(mp), "r"(p.x0), "r"(p.y0), "r"(0), "r"(0), "r"(b) : "memory");
  }
  asm volatile("{\n .reg .pred P1;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n" :: "r"(b) : "memory");
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) p.out[i] = reinterpret_cast<float*>(sm)[i];
}
int main(int argc, char** argv) {
  int use_global = argc > 1 ? atoi(argv[1]) : 0;
  int neg = argc > 2 ? atoi(argv[2]) : 1;
  int bw = argc > 3 ? atoi(argv[3]) : 12;
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  const int W = 8, H = 8, C = 8, N = 4;
  std::vector<float> hx(W*H*C*N); for (size_t i = 0; i < hx.size(); ++i) hx[i] = (float)i;
  float *dx, *dout; cudaMalloc(&dx, hx.size()*4); cudaMemcpy(dx, hx.data(), hx.size()*4, cudaMemcpyHostToDevice);
  P p; cuuint64_t dims[4] = {W, H, C, N}; cuuint64_t str[3] = {W*4, W*H*4, (cuuint64_t)W*H*C*4};
  cuuint32_t box[4] = {(cuuint32_t)bw, 10, 2, 4}; cuuint32_t es[4] = {1,1,1,1};
  CUresult r = enc(&p.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* dm; cudaMalloc(&dm, sizeof(CUtensorMap)); cudaMemcpy(dm, &p.m, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  p.gm = dm; p.use_global = use_global; p.x0 = (neg & 1) ? -1 : 0; p.y0 = (neg & 2) ? -1 : 0;
  p.n = bw*10*2*4; cudaMalloc(&dout, p.n*4); p.out = dout;
  k<<<1, 128, p.n*4>>>(p);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ho(p.n); cudaMemcpy(ho.data(), dout, p.n*4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int n = 0; n < 4; ++n) for (int c = 0; c < 2; ++c) for (int y = 0; y < 10; ++y) for (int x = 0; x < bw; ++x) {
    int gx = x + p.x0, gy = y + p.y0; float want = (gx >= 0 && gx < W && gy >= 0 && gy < H && n < N) ? hx[((n*C + c)*H + gy)*W + gx] : 0.f;
    if (ho[((n*2 + c)*10 + y)*bw + x] != want) ++bad;
  }
  printf("global=%d neg=%d bw=%d encode=%d kernel=%s mismatches=%d\n", use_global, neg, bw, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
