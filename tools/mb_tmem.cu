// Microbenchmark (debug tool): tcgen05.ld (TMEM -> registers) throughput on
// B200, to judge TMEM as a second operand store next to shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmem tools/mb_tmem.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int iters, float* out) {
    __shared__ unsigned taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(&taddr_s);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = taddr_s + ((unsigned)(32 * (warp % 4)) << 16);
    // fill 256 columns with lane-dependent data
    for (int c = 0; c < 256; c += 8) {
        float v = threadIdx.x * 1e-3f + c;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c),
                     "f"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        float r[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned a = base + (unsigned)(((it * 4 + u) * 8 + warp * 24) & 255);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(r[u][0]), "=f"(r[u][1]), "=f"(r[u][2]), "=f"(r[u][3]), "=f"(r[u][4]),
                           "=f"(r[u][5]), "=f"(r[u][6]), "=f"(r[u][7])
                         : "r"(a));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += r[u][j];
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr_s));
}

// conv-like inner loop: per tap one tcgen05.ld of TH consecutive columns at a
// warp-uniform (data-dependent) column, then TH FMUL+FADD pairs
struct Tap { float v; int col; };
template <int NW, int TH, int KW>
__global__ void __launch_bounds__(NW * 32, 1) kc(const Tap* taps, int ntaps, int reps, float* out) {
    __shared__ unsigned taddr_s;
    __shared__ Tap ts[KW * 256];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(&taddr_s);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < KW * ntaps; i += blockDim.x) ts[i] = taps[(warp % 2) * 0 + i];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = taddr_s + ((unsigned)(32 * (warp % 4)) << 16);
    for (int c = 0; c < 512; c += 8) {
        float v = threadIdx.x * 1e-3f + c;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c), "f"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    float acc[KW][TH];
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < TH; ++j) acc[a][j] = 0.f;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const Tap* seg = ts + kk * ntaps;
#pragma unroll 4
            for (int t = 0; t < ntaps; ++t) {
                const Tap tp = seg[t];
                float x[TH];
                if constexpr (TH == 8) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]),
                                   "=f"(x[7])
                                 : "r"(base + tp.col));
                } else {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                                 : "r"(base + tp.col));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < TH; ++j) acc[kk][j] = __fadd_rn(acc[kk][j], __fmul_rn(tp.v, x[j]));
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < TH; ++j) s += acc[a][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int NW, int TH, int KW>
void runc(int ntaps, int reps, int colstep) {
    Tap h[KW * 256];
    for (int i = 0; i < KW * ntaps; ++i) h[i] = Tap{1e-3f * (i % 13), (i * colstep) % (512 - TH)};
    Tap* d;
    float* o;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * NW * 32 * 4);
    kc<NW, TH, KW><<<148, NW * 32>>>(d, ntaps, 1, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kc<NW, TH, KW><<<148, NW * 32>>>(d, ntaps, reps, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = 148.0 * NW * 32 * reps * KW * ntaps * TH;
    printf("conv-loop NW=%d TH=%d KW=%d colstep=%d: %.3f ms  %.2f TMAC/s  err=%s\n", NW, TH, KW, colstep, ms,
           macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(o);
}

template <int NW>
void run(int iters) {
    float* o;
    cudaMalloc(&o, 148 * NW * 32 * 4);
    k<NW><<<148, NW * 32>>>(10, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<NW><<<148, NW * 32>>>(iters, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * NW * iters * 4 * 1024;  // 4 loads x (32 lanes x 8 cols x 4 B) per warp-iteration
    printf("warps/SM=%d: %.3f ms  TMEM read %.1f TB/s  = %.1f B/clk/SM @1.965GHz  err=%s\n", NW, ms, bytes / ms / 1e9,
           bytes / ms / 1e-3 / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(o);
}

int main() {
    run<4>(20000);
    run<8>(20000);
    run<16>(10000);
    runc<8, 8, 8>(64, 200, 8);
    runc<16, 8, 8>(64, 100, 8);
    runc<16, 8, 4>(64, 200, 8);
    runc<16, 8, 4>(64, 200, 1);   // unaligned columns
    runc<16, 8, 4>(64, 200, 3);
    runc<32, 8, 4>(64, 100, 1);
    return 0;
}
