// Unit probe (debug tool) for the TMA -> tcgen05.cp path of csrc/tmc.cuh:
// step 1 TMA box into shared memory, step 2 tcgen05.cp.32x128b.warpx4 into
// TMEM, step 3 tcgen05.ld back; prints the first mismatches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2011_06295_b200/csrc \
//        -o tools/tmc_unit tools/tmc_unit.cu -lcuda
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tmc.cuh"

using namespace scb;

struct UParams {
    CUtensorMap tmap;
    float* out_smem;  // [6 rows][32 n][4]
    float* out_tmem;  // [128 lanes][24 cols]
    int step;
};

__global__ void k_unit(const __grid_constant__ UParams p) {
    __shared__ __align__(1024) float buf[6 * 32 * 4];
    __shared__ uint64_t bar, cbar;
    __shared__ unsigned taddr;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&cbar, 1);
#ifndef NO_MBINIT_FENCE
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (p.step == 0) goto out;
    if (tid == 0) {
        mbar_arrive_tx(&bar, sizeof(buf));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(buf)),
            "l"(&p.tmap), "r"(-1), "r"(0), "r"(-1), "r"(0), "r"(smem_u32(&bar))
            : "memory");
        mbar_wait(&bar, 0);
        if (p.step >= 2) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int h = 0; h < 6; ++h)
                asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr + 4 * h),
                             "l"(tmc_desc(smem_u32(buf + h * 128), 128))
                             : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&cbar))
                         : "memory");
            mbar_wait(&cbar, 0);
        }
    }
    __syncthreads();
    for (int i = tid; i < 6 * 32 * 4; i += blockDim.x) p.out_smem[i] = buf[i];
    if (p.step >= 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float v[16];
        tmi_ld<16>(v, taddr + ((unsigned)(32 * (warp & 3)) << 16));
        tmi_wait<16>(v);
        for (int j = 0; j < 16; ++j) p.out_tmem[(32 * (warp & 3) + lane) * 24 + j] = v[j];
        float w[8];
        tmi_ld<8>(w, taddr + 16 + ((unsigned)(32 * (warp & 3)) << 16));
        tmi_wait<8>(w);
        for (int j = 0; j < 8; ++j) p.out_tmem[(32 * (warp & 3) + lane) * 24 + 16 + j] = w[j];
    }
out:
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

int main() {
    const int N = 32, C = 2, W = 4;
    std::vector<float> x(N * C * W * W);
    for (size_t i = 0; i < x.size(); ++i) x[i] = (float)i;
    float *dx, *ds, *dt;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&ds, 6 * 32 * 4 * 4);
    cudaMalloc(&dt, 128 * 24 * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    UParams p{};
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)N, (cuuint64_t)W, (cuuint64_t)C};
    cuuint64_t strides[3] = {(cuuint64_t)C * W * W * 4, (cuuint64_t)W * 4, (cuuint64_t)W * W * 4};
    cuuint32_t box[4] = {4, 32, 6, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const char* mode = getenv("TMODE");
    if (mode && mode[0] == 'n') {  // natural order (w, h, c, n)
        dims[1] = W; dims[2] = C; dims[3] = N;
        strides[0] = W * 4; strides[1] = W * W * 4; strides[2] = (cuuint64_t)C * W * W * 4;
        box[1] = 6; box[2] = 1; box[3] = 32;
    }
    CUresult cr = enc(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)cr);
    p.out_smem = ds;
    p.out_tmem = dt;
    for (int step = 0; step <= 2; ++step) {
        p.step = step;
        k_unit<<<1, 128>>>(p);
        cudaError_t e = cudaDeviceSynchronize();
        printf("step %d: %s\n", step, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        if (step == 0) continue;
        std::vector<float> s(6 * 32 * 4), t(128 * 24);
        cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(t.data(), dt, t.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int h = 0; h < 6; ++h)
            for (int n = 0; n < 32; ++n)
                for (int w = 0; w < 4; ++w) {
                    const int gy = h - 1, gx = w - 1;
                    const float want = (gy < 0 || gy >= W || gx < 0 || gx >= W) ? 0.f : x[(n * C + 0) * 16 + gy * 4 + gx];
                    const float got = s[(h * 32 + n) * 4 + w];
                    if (got != want && bad++ < 5) printf("  smem h%d n%d w%d got %g want %g\n", h, n, w, got, want);
                    if (step == 2)
                        for (int qq = 0; qq < 4; ++qq) {
                            const float gt = t[(32 * qq + n) * 24 + h * 4 + w];
                            if (gt != want && bad++ < 10) printf("  tmem q%d h%d n%d w%d got %g want %g\n", qq, h, n, w, gt, want);
                        }
                }
        printf("step %d bad %d\n", step, bad);
    }
    return 0;
}
