// sm_100a kernels: the generic (any geometry / ragged / f64) direct sparse
// conv and the 2x2 max-pool glue.  The register-tiled kernel lives in
// tiled.cuh and is instantiated by the generated inst_gen_*.cu units.
#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"
#include "variants.h"

namespace scb {

// ------------------------------------------------------------------------
// generic kernel: any geometry / stride / ragged CSR / f64.
// One thread per output element; consecutive threads walk f then e of the
// same (n, k) plane, so the tap stream of a warp is (mostly) uniform.
// ------------------------------------------------------------------------
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_generic(const __grid_constant__ GenericParams p) {
    const T* __restrict__ x = static_cast<const T*>(p.x);
    const T* __restrict__ vals = static_cast<const T*>(p.values);
    T* __restrict__ y = static_cast<T*>(p.y);
    const int64_t total = (int64_t)p.n * p.k * p.e * p.f;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)(idx % p.f);
        int64_t t = idx / p.f;
        const int e = (int)(t % p.e);
        t /= p.e;
        const int k = (int)(t % p.k);
        const int64_t n = t / p.k;
        const int y0 = e * p.stride - p.pad, x0 = f * p.stride - p.pad;
        const T* xn = x + n * p.c * p.h * p.w;
        const int t0 = p.rowptr[k], t1 = p.rowptr[k + 1];
        if constexpr (std::is_same<T, double>::value) {
            double acc = p.bias ? static_cast<const double*>(p.bias)[k] : 0.0;
            for (int q = t0; q < t1; ++q) {
                const int d = p.dec[q];
                const int c = d / (p.kr * p.ks), rs = d - c * (p.kr * p.ks);
                const int gy = y0 + rs / p.ks, gx = x0 + rs % p.ks;
                double xv = 0.0;
                if (gy >= 0 && gy < p.h && gx >= 0 && gx < p.w) xv = xn[((int64_t)c * p.h + gy) * p.w + gx];
                if constexpr (MODE == MODE_EXACT) acc = __dadd_rn(acc, __dmul_rn(vals[q], xv));
                else acc = __fma_rn(vals[q], xv, acc);
            }
            if ((p.flags & SCB_FLAG_RELU) && acc < 0.0) acc = 0.0;
            y[idx] = acc;
        } else {
            float acc = 0.f;
            if (p.bias) acc = static_cast<const float*>(p.bias)[k];  // compute dtype
            for (int q = t0; q < t1; ++q) {
                const int d = p.dec[q];
                const int c = d / (p.kr * p.ks), rs = d - c * (p.kr * p.ks);
                const int gy = y0 + rs / p.ks, gx = x0 + rs % p.ks;
                float xv = 0.f, v;
                if constexpr (std::is_same<T, __half>::value) {
                    if (gy >= 0 && gy < p.h && gx >= 0 && gx < p.w)
                        xv = __half2float(xn[((int64_t)c * p.h + gy) * p.w + gx]);
                    v = __half2float(vals[q]);
                    acc = __fmaf_rn(v, xv, acc);  // f16*f16 is exact in f32
                } else {
                    if (gy >= 0 && gy < p.h && gx >= 0 && gx < p.w) xv = xn[((int64_t)c * p.h + gy) * p.w + gx];
                    v = vals[q];
                    acc = mac1<MODE>(acc, v, xv);
                }
            }
            if (p.flags & SCB_FLAG_RELU) acc = relu_io<T>(acc);  // f16: round, then max(., 0)
            if constexpr (std::is_same<T, __half>::value) y[idx] = __float2half_rn(acc);
            else y[idx] = acc;
        }
    }
}

template <typename T, int MODE>
static cudaError_t launch_generic_t(const GenericParams& p, cudaStream_t st) {
    const int64_t total = (int64_t)p.n * p.k * p.e * p.f;
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    k_generic<T, MODE><<<(unsigned)blocks, 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_generic(const GenericParams& p, int dtype, bool fast, cudaStream_t st) {
    if (dtype == SCB_F64) return fast ? launch_generic_t<double, MODE_FMA>(p, st) : launch_generic_t<double, MODE_EXACT>(p, st);
    if (dtype == SCB_F16) return launch_generic_t<__half, MODE_FMA>(p, st);
    return fast ? launch_generic_t<float, MODE_FMA>(p, st) : launch_generic_t<float, MODE_EXACT>(p, st);
}

// ------------------------------------------------------------------------
// 2x2/2 max pool glue
// ------------------------------------------------------------------------
template <typename T>
__global__ void k_maxpool2(const T* __restrict__ x, T* __restrict__ y, int64_t planes, int h, int w) {
    const int ho = h >> 1, wo = w >> 1;
    const int64_t total = planes * ho * wo;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int ox = (int)(i % wo);
        int64_t t = i / wo;
        const int oy = (int)(t % ho);
        const int64_t pl = t / ho;
        const T* b = x + (pl * h + 2 * oy) * w + 2 * ox;
        float a0, a1, a2, a3;
        if constexpr (std::is_same<T, __half>::value) {
            a0 = __half2float(b[0]); a1 = __half2float(b[1]); a2 = __half2float(b[w]); a3 = __half2float(b[w + 1]);
            y[i] = __float2half_rn(fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        } else {
            y[i] = (T)fmax(fmax((double)b[0], (double)b[1]), fmax((double)b[w], (double)b[w + 1]));
        }
    }
}

// Activation fake-quant pass (quantize.py:332-338) over `count` activations in place.
template <typename T>
__global__ void k_fake_quant(T* y, int64_t count, const ActQuant q) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        if constexpr (std::is_same<T, __half>::value) y[i] = fq_f16(y[i], q);
        else if constexpr (std::is_same<T, double>::value) y[i] = fq_f64(y[i], q);
        else y[i] = fq_f32(y[i], q);
    }
}

cudaError_t launch_fake_quant(int dtype, void* y, int64_t count, const ActQuant& q, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (dtype == SCB_F16)
        k_fake_quant<__half><<<(unsigned)blocks, 256, 0, st>>>((__half*)y, count, q);
    else if (dtype == SCB_F64)
        k_fake_quant<double><<<(unsigned)blocks, 256, 0, st>>>((double*)y, count, q);
    else
        k_fake_quant<float><<<(unsigned)blocks, 256, 0, st>>>((float*)y, count, q);
    return cudaGetLastError();
}

cudaError_t launch_maxpool2(int dtype, const void* x, void* y, int64_t planes, int h, int w, cudaStream_t st) {
    const int64_t total = planes * (h >> 1) * (w >> 1);
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (dtype == SCB_F16)
        k_maxpool2<__half><<<(unsigned)blocks, 256, 0, st>>>((const __half*)x, (__half*)y, planes, h, w);
    else if (dtype == SCB_F64)
        k_maxpool2<double><<<(unsigned)blocks, 256, 0, st>>>((const double*)x, (double*)y, planes, h, w);
    else
        k_maxpool2<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)x, (float*)y, planes, h, w);
    return cudaGetLastError();
}

// 32 x 32 tiles through shared memory (33-word rows: no bank conflicts), 8 rows per thread
template <typename T>
__global__ void __launch_bounds__(256) k_transpose(const T* __restrict__ x, int64_t ldx, T* __restrict__ y, int64_t ldy,
                                                   int64_t rows, int64_t cols) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t r = r0 + ty + k, c = c0 + tx;
        if (r < rows && c < cols) tile[ty + k][tx] = x[r * ldx + c];
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t c = c0 + ty + k, r = r0 + tx;
        if (r < rows && c < cols) y[c * ldy + r] = tile[tx][ty + k];
    }
}

cudaError_t launch_transpose(int es, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t rows, int64_t cols,
                             cudaStream_t st) {
    const int64_t gx = (cols + 31) / 32, gy = (rows + 31) / 32;
    if (gy > 65535 || gx > 0x7fffffffLL) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)gx, (unsigned)gy);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (es == 4)
        e = cudaLaunchKernelEx(&cfg, k_transpose<float>, static_cast<const float*>(x), ldx, static_cast<float*>(y), ldy,
                               rows, cols);
    else if (es == 2)
        e = cudaLaunchKernelEx(&cfg, k_transpose<unsigned short>, static_cast<const unsigned short*>(x), ldx,
                               static_cast<unsigned short*>(y), ldy, rows, cols);
    else
        e = cudaLaunchKernelEx(&cfg, k_transpose<double>, static_cast<const double*>(x), ldx, static_cast<double*>(y),
                               ldy, rows, cols);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace scb
