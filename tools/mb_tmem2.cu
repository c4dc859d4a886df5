// Microbenchmark (debug tool): the tap loop of the TMEM image-lane kernel
// (csrc/tmi.cuh).  Per tap: one warp-uniform {value, column} from shared
// memory, one tcgen05.ld.32x32b.x{WIN} of the lane's window at that column,
// WIN exact FMUL+FADD pairs; the load of tap t+1 is in flight while tap t is
// multiplied (ping-pong register windows, tcgen05.wait::ld ties them).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmem2 tools/mb_tmem2.cu
#include <cuda_runtime.h>

#include <cstdio>

struct Tap {
    float v;
    unsigned col;
};

template <int N>
struct Win {
    float x[N];
};

template <int N>
__device__ __forceinline__ void ldtm(Win<N>& w, unsigned a);
template <>
__device__ __forceinline__ void ldtm<16>(Win<16>& w, unsigned a) {
    float* x = w.x;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15])
        : "r"(a));
}
template <int N>
__device__ __forceinline__ void waitld(Win<N>& w);
template <>
__device__ __forceinline__ void waitld<16>(Win<16>& w) {
    float* x = w.x;
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]), "+f"(x[4]), "+f"(x[5]), "+f"(x[6]), "+f"(x[7]),
                   "+f"(x[8]), "+f"(x[9]), "+f"(x[10]), "+f"(x[11]), "+f"(x[12]), "+f"(x[13]), "+f"(x[14]),
                   "+f"(x[15])::"memory");
}

// empty volatile asm that "modifies" the accumulators: orders the MAC block
// after the preceding (volatile) tcgen05.ld so the load overlaps the MACs
template <int N>
__device__ __forceinline__ void pin(float (&a)[N]) {
#pragma unroll
    for (int j = 0; j < N; j += 8)
        asm volatile("" : "+f"(a[j]), "+f"(a[j + 1]), "+f"(a[j + 2]), "+f"(a[j + 3]), "+f"(a[j + 4]), "+f"(a[j + 5]),
                     "+f"(a[j + 6]), "+f"(a[j + 7]));
}

template <int N>
__device__ __forceinline__ void mac(float (&acc)[N], float v, const Win<N>& w) {
#pragma unroll
    for (int j = 0; j < N; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(v, w.x[j]));
}

// NW warps per CTA (NW/4 per TMEM lane quarter), KW output channels per warp,
// each with nt taps per rep
template <int NW, int KW, int WIN, bool PIPE>
__global__ void __launch_bounds__(NW * 32, 1) kc(const Tap* taps, int nt, int reps, float* out) {
    __shared__ unsigned taddr_s;
    __shared__ Tap ts[NW][KW][64];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < NW * KW * 64; i += blockDim.x) (&ts[0][0][0])[i] = taps[i % (KW * 64)];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = taddr_s + ((unsigned)(32 * (warp % 4)) << 16);
    for (int c = 0; c < 512; c += 16) {
        float v = threadIdx.x * 1e-3f + c;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                base + c),
            "f"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    float acc[KW][WIN];
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < WIN; ++j) acc[a][j] = 0.f;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const Tap* seg = ts[warp][kk];
            Win<WIN> xa, xb;
            Tap ta = seg[0];
            ldtm(xa, base + ta.col);
            waitld(xa);
            int t = 0;
            for (; t + 2 <= nt; t += 2) {
                const Tap tb = seg[t + 1];
                ldtm(xb, base + tb.col);
                if (PIPE) pin(acc[kk]);
                mac(acc[kk], ta.v, xa);
                waitld(xb);
                ta = seg[t + 2];  // seg has a sentinel beyond nt
                ldtm(xa, base + ta.col);
                if (PIPE) pin(acc[kk]);
                mac(acc[kk], tb.v, xb);
                waitld(xa);
            }
            if (t < nt) mac(acc[kk], ta.v, xa);
        }
    }
    float s = 0;
#pragma unroll
    for (int a = 0; a < KW; ++a)
#pragma unroll
        for (int j = 0; j < WIN; ++j) s += acc[a][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int NW, int KW, int WIN, bool PIPE>
void runc(int nt, int reps) {
    Tap h[KW * 64];
    for (int i = 0; i < KW * 64; ++i) h[i] = Tap{1e-3f * (i % 13), (unsigned)((i * 7) % (512 - WIN))};
    Tap* d;
    float* o;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * NW * 32 * 4);
    kc<NW, KW, WIN, PIPE><<<148, NW * 32>>>(d, nt, 1, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kc<NW, KW, WIN, PIPE><<<148, NW * 32>>>(d, nt, reps, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = 148.0 * NW * 32 * reps * KW * nt * WIN;
    printf("tap-loop PIPE=%d NW=%d KW=%d WIN=%d nt=%d: %.3f ms  %.2f TMAC/s (%.0f%% of 18.0)  err=%s\n", (int)PIPE, NW, KW, WIN, nt, ms,
           macs / ms / 1e9, macs / ms / 1e9 / 18.04 * 100, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(o);
}

int main() {
#define BOTH(NW, KW, NT, REPS) runc<NW, KW, 16, false>(NT, REPS); runc<NW, KW, 16, true>(NT, REPS);
    BOTH(8, 1, 62, 400)
    BOTH(16, 1, 62, 200)
    BOTH(32, 1, 62, 100)
    BOTH(8, 2, 62, 200)
    BOTH(16, 2, 62, 100)
    BOTH(16, 4, 62, 50)
    BOTH(16, 1, 4, 3000)
    BOTH(32, 1, 4, 1500)
    BOTH(16, 2, 3, 2000)
    return 0;
}
