// Microbenchmark (debug tool): the direct kernel's inner tap loop in
// isolation -- input tile and tap list resident in shared memory, no staging,
// no barriers -- to separate the loop's own throughput from the pipeline.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_direct tools/mb_direct.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

struct __align__(8) Tap { float v; int off; };

template <int V> struct VT;
template <> struct VT<1> { using T = float; };
template <> struct VT<2> { using T = float2; };
template <> struct VT<4> { using T = float4; };

template <int TH, int KW, int MODE, int V = 1>
__global__ void __launch_bounds__(256, 2) k(const Tap* taps, int ntaps, int reps, float* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    float* xs = reinterpret_cast<float*>(sm);
    Tap* ts = reinterpret_cast<Tap*>(sm + 40960);
    for (int i = threadIdx.x; i < 10240; i += blockDim.x) xs[i] = 1.0f + (i & 7) * 1e-3f;
    for (int i = threadIdx.x; i < ntaps * KW; i += blockDim.x) ts[i] = taps[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float acc[KW][TH * V];
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < TH * V; ++j) acc[a][j] = 0.f;
    const char* xl = reinterpret_cast<const char*>(xs + lane * V + warp * 8);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const Tap* seg = ts + kk * ntaps;
#pragma unroll 4
            for (int t = 0; t < ntaps; ++t) {
                const Tap tp = seg[t];
                const float* xp = reinterpret_cast<const float*>(xl + tp.off);
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    const typename VT<V>::T xv = *reinterpret_cast<const typename VT<V>::T*>(xp + j * 160);
                    const float* xf = reinterpret_cast<const float*>(&xv);
#pragma unroll
                    for (int u = 0; u < V; ++u) {
                        if (MODE == 0) acc[kk][j * V + u] = __fadd_rn(acc[kk][j * V + u], __fmul_rn(tp.v, xf[u]));
                        else acc[kk][j * V + u] = __fmaf_rn(tp.v, xf[u], acc[kk][j * V + u]);
                    }
                }
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < TH * V; ++j) s += acc[a][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int TH, int KW, int MODE, int V = 1>
void run(int ntaps, int reps) {
    std::vector<Tap> h(ntaps * KW);
    for (int i = 0; i < ntaps * KW; ++i) h[i] = Tap{1e-3f * (i % 13), 16 * ((i * 37) % 300)};
    Tap* d; float* o;
    cudaMalloc(&d, h.size() * sizeof(Tap));
    cudaMemcpy(d, h.data(), h.size() * sizeof(Tap), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    auto kern = k<TH, KW, MODE, V>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int grid = 148 * 2;
    kern<<<grid, 256, 100 * 1024>>>(d, ntaps, 1, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, 256, 100 * 1024>>>(d, ntaps, reps, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double macs = (double)grid * 256 * reps * KW * ntaps * TH * V;
    printf("TH=%d KW=%d V=%d mode=%s ntaps=%d: %.3f ms  %.2f TMAC/s  err=%s\n", TH, KW, V, MODE ? "ffma" : "mul+add",
           ntaps, ms, macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(o);
}

int main() {
    run<8, 8, 0, 1>(64, 200);
    run<8, 4, 0, 2>(64, 200);
    run<4, 4, 0, 4>(64, 200);
    run<8, 2, 0, 4>(64, 200);
    run<4, 4, 1, 4>(64, 200);
    return 0;
}
