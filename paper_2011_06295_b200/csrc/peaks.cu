// CUDA-core arithmetic throughput probes (the FMA roofline denominators the
// north star asks for; MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// Each probe runs 8 independent chains per thread over a full grid and
// reports multiply-accumulates per second.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "common.h"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) k_probe(float a, float b, float* out) {
    float acc[kChains], x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) { acc[i] = a * (threadIdx.x + i); x[i] = b + i; }
    float v = a + b;
    for (int it = 0; it < kIters; ++it) {
        // the multiplicand rotates through the chains so products cannot be hoisted
#pragma unroll
        for (int i = 0; i < kChains; ++i) x[i] = acc[(i + 1) % kChains];
#pragma unroll
        for (int i = 0; i < kChains; i += 2) {
            if constexpr (OP == 0) {  // FFMA
                acc[i] = __fmaf_rn(v, x[i], acc[i]);
                acc[i + 1] = __fmaf_rn(v, x[i + 1], acc[i + 1]);
            } else if constexpr (OP == 1) {  // FFMA2
                unsigned long long A, X, V, R;
                asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(acc[i]), "f"(acc[i + 1]));
                asm("mov.b64 %0, {%1,%2};" : "=l"(X) : "f"(x[i]), "f"(x[i + 1]));
                asm("mov.b64 %0, {%1,%1};" : "=l"(V) : "f"(v));
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(R) : "l"(X), "l"(V), "l"(A));
                asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(R));
            } else if constexpr (OP == 2) {  // FMUL + FADD
                acc[i] = __fadd_rn(acc[i], __fmul_rn(v, x[i]));
                acc[i + 1] = __fadd_rn(acc[i + 1], __fmul_rn(v, x[i + 1]));
            } else if constexpr (OP == 3) {  // FMUL2 + 2 FADD
                unsigned long long X, V, P;
                asm("mov.b64 %0, {%1,%2};" : "=l"(X) : "f"(x[i]), "f"(x[i + 1]));
                asm("mov.b64 %0, {%1,%1};" : "=l"(V) : "f"(v));
                asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(P) : "l"(X), "l"(V));
                float p0, p1;
                asm("mov.b64 {%0,%1}, %2;" : "=f"(p0), "=f"(p1) : "l"(P));
                acc[i] = __fadd_rn(acc[i], p0);
                acc[i + 1] = __fadd_rn(acc[i + 1], p1);
            } else if constexpr (OP == 4) {  // 2 FMUL + FADD2
                float p0 = __fmul_rn(v, x[i]), p1 = __fmul_rn(v, x[i + 1]);
                unsigned long long A, P, R;
                asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(acc[i]), "f"(acc[i + 1]));
                asm("mov.b64 %0, {%1,%2};" : "=l"(P) : "f"(p0), "f"(p1));
                asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(P));
                asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(R));
            } else if constexpr (OP == 5) {  // FHFMA (f16 x f16 + f32)
                __half hv = __float2half_rn(v), h0 = __float2half_rn(x[i]), h1 = __float2half_rn(x[i + 1]);
                unsigned short uv = __half_as_ushort(hv), u0 = __half_as_ushort(h0), u1 = __half_as_ushort(h1);
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(u0), "h"(uv));
                asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i + 1]) : "h"(u1), "h"(uv));
            } else {  // HFMA2
                __half2 A = __floats2half2_rn(acc[i], acc[i + 1]);
                __half2 X = __floats2half2_rn(x[i], x[i + 1]);
                __half2 V = __float2half2_rn(v);
#pragma unroll
                for (int u = 0; u < 4; ++u) A = __hfma2(V, X, A);
                float2 f = __half22float2(A);
                acc[i] = f.x; acc[i + 1] = f.y;
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += acc[i];
    if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int OP>
double run_probe(int* err) {
    const int blocks = 148 * 8, threads = 256;
    float* d_out = nullptr;
    cudaMalloc(&d_out, 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_probe<OP><<<blocks, threads>>>(1.0001f, 0.5f, d_out);  // warm-up
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_probe<OP><<<blocks, threads>>>(1.0001f, 0.5f, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) *err = 1;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_out);
    double macs_per_thread = (double)kIters * kChains * (OP == 6 ? 4 : 1);
    double total = macs_per_thread * blocks * threads * reps;
    return total / (ms * 1e-3);
}

}  // namespace

extern "C" SCB_API scb_status scb_fma_peaks(int32_t device, char* names, double* macs_per_s, int32_t cap,
                                            int32_t* count) {
    if (!names || !macs_per_s || !count) return scb::fail(SCB_ERR_ARG, "NULL");
    if (cudaSetDevice(device) != cudaSuccess) return scb::fail(SCB_ERR_CUDA, "cudaSetDevice");
    const char* nm[] = {"ffma", "ffma2", "fmul_fadd", "fmul2_fadd", "fmul_fadd2", "fhfma", "hfma2"};
    int err = 0;
    double v[7];
    v[0] = run_probe<0>(&err);
    v[1] = run_probe<1>(&err);
    v[2] = run_probe<2>(&err);
    v[3] = run_probe<3>(&err);
    v[4] = run_probe<4>(&err);
    v[5] = run_probe<5>(&err);
    v[6] = run_probe<6>(&err);
    if (err) return scb::fail(SCB_ERR_CUDA, "probe kernel failed");
    int n = cap < 7 ? cap : 7;
    for (int i = 0; i < n; ++i) {
        std::memset(names + 16 * i, 0, 16);
        std::strncpy(names + 16 * i, nm[i], 15);
        macs_per_s[i] = v[i];
    }
    *count = n;
    return SCB_OK;
}
