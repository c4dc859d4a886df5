// Standalone harness for the TMEM image-lane kernel (csrc/tmi.cuh): random
// unified-sparse taps for one VGG-CIFAR geometry, device-timed launches, and
// (with -DTMI_TRACE) per-stage clock64 stamps of CTA 0's filler and first
// consumer.  Debug tool; the library path is tested by tools/probe_tmi.py.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2011_06295_b200/csrc \
//        [-DTMI_TRACE] -o tools/tmi_harness tools/tmi_harness.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#ifdef TMI_TRACE
__device__ long long g_trace[2][4096][6];
#define TMI_STAMP(role, s, i) \
    do { if (blockIdx.x == 0 && lane == 0 && (s) < 4096) g_trace[role][s][i] = clock64(); } while (0)
#endif
#include "tmc.cuh"
#include "tmr.cuh"
#include "tmi.cuh"
#include <cudaTypedefs.h>

using namespace scb;

template <int W, int TE, int J, int KW, int WQ>
void run(int N, int C, int K, int L, int depth, int reps) {
    using G = TmiGeom<W, TE, J>;
    const int HW = W * W;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd;
    std::vector<float> x((size_t)N * C * HW);
    for (auto& v : x) v = nd(rng);
    const int nst = (C + G::CS - 1) / G::CS;
    std::vector<TmiTap> taps;
    std::vector<int32_t> tb(K + 1), so((size_t)K * (nst + 1));
    int tcap = 2;
    for (int k = 0; k < K; ++k) {
        tb[k] = (int)taps.size();
        std::vector<int> idx(C * 9);
        for (int i = 0; i < C * 9; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), rng);
        idx.resize(L);
        std::sort(idx.begin(), idx.end());
        int st = 0;
        for (int t = 0; t < L; ++t) {
            const int c = idx[t] / 9, r = idx[t] % 9 / 3, s = idx[t] % 3;
            while (st <= nst && st * G::CS <= c) so[(size_t)k * (nst + 1) + st++] = t;
            taps.push_back(TmiTap{nd(rng), (uint32_t)((c % G::CS) * G::SW + (s * G::CPR + r) * G::RW)});
        }
        while (st <= nst) so[(size_t)k * (nst + 1) + st++] = L;
        if (taps.size() & 1) taps.push_back(TmiTap{0.f, 0u});
        tcap = std::max(tcap, (int)taps.size() - tb[k]);
    }
    tb[K] = (int)taps.size();
    float *dx, *dy;
    TmiTap* dt;
    int32_t *dtb, *dso;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dy, (size_t)N * K * HW * 4);
    cudaMalloc(&dt, taps.size() * sizeof(TmiTap));
    cudaMalloc(&dtb, tb.size() * 4);
    cudaMalloc(&dso, so.size() * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, taps.data(), taps.size() * sizeof(TmiTap), cudaMemcpyHostToDevice);
    cudaMemcpy(dtb, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dso, so.data(), so.size() * 4, cudaMemcpyHostToDevice);
    int ip = (G::CS * HW + 3) / 4 * 4;
    while ((ip / 4) % 2 == 0) ip += 4;
    const int stage_fl = (G::IMGS * ip + 31) / 32 * 32;
    const int cap = 4 * WQ * KW;
    const size_t smem = (size_t)4 * depth * stage_fl * 4 + (size_t)cap * tcap * 8 + (size_t)cap * (nst + 1) * 4;
    TmiParams p{};
    p.x = dx; p.y = dy; p.bias = nullptr; p.taps = dt; p.tbase = dtb; p.soff = dso;
    p.n = N; p.c = C; p.k = K; p.nst = nst; p.nblk = (N + G::IMGS - 1) / G::IMGS; p.depth = depth;
    p.ipitch = ip; p.stage_fl = stage_fl; p.tcap = tcap; p.items = p.nblk * K; p.flags = SCB_FLAG_NO_PDL;
    const unsigned grid = std::min(148, p.items);
    cudaError_t e = launch_tmi_t<W, TE, J, KW, WQ, 0>(p, grid, smem, 0);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch_tmi_t<W, TE, J, KW, WQ, 0>(p, grid, smem, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = (double)N * K * HW * L;
    printf("W=%d TE=%d J=%d KW=%d WQ=%d depth=%d CS=%d NSET=%d smem=%zu: %.1f us  %.2f TMAC/s (%.2f of 18.0)  %s/%s\n",
           W, TE, J, KW, WQ, depth, G::CS, G::NSET, smem, ms / reps * 1e3, macs / (ms / reps * 1e-3) / 1e12,
           macs / (ms / reps * 1e-3) / 1e12 / 18.04, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
#ifdef TMI_TRACE
    static long long tr[2][4096][6];
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
    const int ns = std::min(nst, 4096);
    for (int role = 0; role < 2; ++role) {
        double d[6] = {0};
        for (int s = 1; s < ns; ++s)
            for (int i = 1; i < 6; ++i) d[i] += (double)(tr[role][s][i] - tr[role][s][i - 1]);
        double per = (double)(tr[role][ns - 1][0] - tr[role][1][0]) / (ns - 2);
        printf("  %s: cycles/stage %.0f; segments", role ? "consumer" : "filler", per);
        for (int i = 1; i < 6; ++i) printf(" %.0f", d[i] / (ns - 1));
        printf("\n");
    }
#endif
    cudaFree(dx); cudaFree(dy); cudaFree(dt); cudaFree(dtb); cudaFree(dso);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    }
    return fn;
}

// TMA -> tcgen05.cp variant (tmc.cuh); CPU check of a sample of outputs (exact mul+add in colidx order)
template <int W, int KW, int WQ>
void run_tmc(int N, int C, int K, int L, int depth, int reps, unsigned extra = 0) {
    using G = TmcGeom<W>;
    const int HW = W * W;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd;
    std::vector<float> x((size_t)N * C * HW);
    for (auto& v : x) v = nd(rng);
    const int nst = (C + G::CS - 1) / G::CS;
    std::vector<TmiTap> taps;
    std::vector<int32_t> tb(K + 1), so((size_t)K * (nst + 1));
    std::vector<std::vector<int>> cidx(K);
    int tcap = 2;
    for (int k = 0; k < K; ++k) {
        tb[k] = (int)taps.size();
        std::vector<int> idx(C * 9);
        for (int i = 0; i < C * 9; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), rng);
        idx.resize(L);
        std::sort(idx.begin(), idx.end());
        cidx[k] = idx;
        int st = 0;
        for (int t = 0; t < L; ++t) {
            const int c = idx[t] / 9, r = idx[t] % 9 / 3, s = idx[t] % 3;
            while (st <= nst && st * G::CS <= c) so[(size_t)k * (nst + 1) + st++] = t;
            taps.push_back(TmiTap{nd(rng), (uint32_t)((c % G::CS) * G::SLOTC + (r - 1) * G::RP + 3 + s)});
        }
        while (st <= nst) so[(size_t)k * (nst + 1) + st++] = L;
        if (taps.size() & 1) taps.push_back(TmiTap{0.f, 0u});
        tcap = std::max(tcap, (int)taps.size() - tb[k]);
    }
    tb[K] = (int)taps.size();
    float *dx, *dy;
    TmiTap* dt;
    int32_t *dtb, *dso;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dy, (size_t)N * K * HW * 4);
    cudaMalloc(&dt, taps.size() * sizeof(TmiTap));
    cudaMalloc(&dtb, tb.size() * 4);
    cudaMalloc(&dso, so.size() * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, taps.data(), taps.size() * sizeof(TmiTap), cudaMemcpyHostToDevice);
    cudaMemcpy(dtb, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dso, so.data(), so.size() * 4, cudaMemcpyHostToDevice);
    TmcParams p{};
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)N, (cuuint64_t)W, (cuuint64_t)C};
    cuuint64_t strides[3] = {(cuuint64_t)C * HW * 4, (cuuint64_t)W * 4, (cuuint64_t)HW * 4};
    cuuint32_t box[4] = {4, (cuuint32_t)G::IMGS, (cuuint32_t)W, (cuuint32_t)G::CS};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult cr = encode_fn()(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int cap = WQ * KW;
    const size_t smem = (size_t)depth * G::SLOT + (size_t)cap * tcap * 8 + (size_t)cap * (nst + 1) * 4;
    p.y = dy; p.bias = nullptr; p.taps = dt; p.tbase = dtb; p.soff = dso;
    p.n = N; p.c = C; p.k = K; p.nst = nst; p.nblk = (N + G::IMGS - 1) / G::IMGS; p.depth = depth;
    p.tcap = tcap; p.items = p.nblk * K; p.flags = SCB_FLAG_NO_PDL | extra;
    const unsigned grid = std::min(148, p.items);
    cudaError_t e = launch_tmc_t<W, KW, WQ, 0>(p, grid, smem, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<float> y((size_t)N * K * HW);
    cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, checked = 0;
    for (int n = 0; n < N; n += 37)
        for (int k = 0; k < K; k += 13)
            for (int e0 = 0; e0 < W; ++e0)
                for (int f0 = 0; f0 < W; ++f0) {
                    float o = 0.f;
                    for (int t = 0; t < L; ++t) {
                        const int c = cidx[k][t] / 9, r = cidx[k][t] % 9 / 3, s = cidx[k][t] % 3;
                        const int yy = e0 + r - 1, xx = f0 + s - 1;
                        const float xv = (yy < 0 || yy >= W || xx < 0 || xx >= W) ? 0.f : x[((size_t)n * C + c) * HW + yy * W + xx];
                        volatile float prod = taps[tb[k] + t].v * xv;
                        o = o + prod;
                    }
                    ++checked;
                    if (o != y[((size_t)n * K + k) * HW + e0 * W + f0]) ++bad;
                }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch_tmc_t<W, KW, WQ, 0>(p, grid, smem, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = (double)N * K * HW * L;
    printf("TMC W=%d KW=%d WQ=%d depth=%d CS=%d NSET=%d smem=%zu enc=%d: %.1f us  %.2f TMAC/s (%.2f of 18.0)  %s/%s/%s  bad %d of %d\n",
           W, KW, WQ, depth, G::CS, G::NSET, smem, (int)cr, ms / reps * 1e3, macs / (ms / reps * 1e-3) / 1e12,
           macs / (ms / reps * 1e-3) / 1e12 / 18.04, cudaGetErrorString(e), cudaGetErrorString(e2),
           cudaGetErrorString(cudaGetLastError()), bad, checked);
#ifdef TMI_TRACE
    static long long tr[2][4096][6];
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
    const int ns = std::min(nst, 4096);
    for (int role = 0; role < 2; ++role) {
        double d[6] = {0};
        for (int s = 1; s < ns; ++s)
            for (int i = 1; i < 6; ++i) d[i] += (double)(tr[role][s][i] - tr[role][s][i - 1]);
        double per = (double)(tr[role][ns - 1][0] - tr[role][1][0]) / (ns - 2);
        printf("  %s: cycles/stage %.0f; segments", role ? "consumer" : "producer", per);
        for (int i = 1; i < 6; ++i) printf(" %.0f", d[i] / (ns - 1));
        printf("\n");
    }
#endif
    cudaFree(dx); cudaFree(dy); cudaFree(dt); cudaFree(dtb); cudaFree(dso);
}

// compact-plane variant (tmr.cuh); CPU check of a sample of outputs (exact mul+add in colidx order)
template <int W, int KW, int WQ>
void run_tmr(int N, int C, int K, int L, int depth, int reps, unsigned extra = 0) {
    using G = TmrGeom<W>;
    const int HW = W * W;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd;
    std::vector<float> x((size_t)N * C * HW);
    for (auto& v : x) v = nd(rng);
    const int nst = (C + G::CS - 1) / G::CS;
    std::vector<TmiTap> taps;
    std::vector<int32_t> tb(K + 1), so((size_t)K * (nst + 1));
    std::vector<std::vector<int>> cidx(K);
    int tcap = 2;
    for (int k = 0; k < K; ++k) {
        tb[k] = (int)taps.size();
        std::vector<int> idx(C * 9);
        for (int i = 0; i < C * 9; ++i) idx[i] = i;
        std::shuffle(idx.begin(), idx.end(), rng);
        idx.resize(L);
        std::sort(idx.begin(), idx.end());
        cidx[k] = idx;
        int st = 0;
        for (int t = 0; t < L; ++t) {
            const int c = idx[t] / 9, r = idx[t] % 9 / 3, s = idx[t] % 3;
            while (st <= nst && st * G::CS <= c) so[(size_t)k * (nst + 1) + st++] = t;
            taps.push_back(TmiTap{nd(rng), (uint32_t)(((c % G::CS) * G::PITCH + (r - 1) * W + (s - 1) + 8) | (s << 16))});
        }
        while (st <= nst) so[(size_t)k * (nst + 1) + st++] = L;
        if (taps.size() & 1) taps.push_back(TmiTap{0.f, 0u});
        tcap = std::max(tcap, (int)taps.size() - tb[k]);
    }
    tb[K] = (int)taps.size();
    float *dx, *dy;
    TmiTap* dt;
    int32_t *dtb, *dso;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dy, (size_t)N * K * HW * 4);
    cudaMalloc(&dt, taps.size() * sizeof(TmiTap));
    cudaMalloc(&dtb, tb.size() * 4);
    cudaMalloc(&dso, so.size() * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, taps.data(), taps.size() * sizeof(TmiTap), cudaMemcpyHostToDevice);
    cudaMemcpy(dtb, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dso, so.data(), so.size() * 4, cudaMemcpyHostToDevice);
    TmcParams p{};
    cuuint64_t dims[3] = {32, (cuuint64_t)N, (cuuint64_t)C / 2};
    cuuint64_t strides[2] = {(cuuint64_t)C * HW * 4, 128};
    cuuint32_t box[3] = {32, 32, (cuuint32_t)G::CS / 2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult cr = encode_fn()(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dx, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int cap = 4 * WQ * KW;
    const size_t smem = 1024 + (size_t)depth * G::SLOT + (size_t)cap * tcap * 8 + (size_t)cap * (nst + 1) * 4;
    p.y = dy; p.bias = nullptr; p.taps = dt; p.tbase = dtb; p.soff = dso;
    p.n = N; p.c = C; p.k = K; p.nst = nst; p.nblk = (N + G::IMGS - 1) / G::IMGS; p.depth = depth;
    p.tcap = tcap; p.items = p.nblk * K; p.flags = SCB_FLAG_NO_PDL | extra;
    const unsigned grid = std::min(148, p.items);
    cudaError_t e = launch_tmr_t<W, KW, WQ, 0>(p, grid, smem, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<float> y((size_t)N * K * HW);
    cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, checked = 0;
    for (int n = 0; n < N; n += 37)
        for (int k = 0; k < K; k += 13)
            for (int e0 = 0; e0 < W; ++e0)
                for (int f0 = 0; f0 < W; ++f0) {
                    float o = 0.f;
                    for (int t = 0; t < L; ++t) {
                        const int c = cidx[k][t] / 9, r = cidx[k][t] % 9 / 3, s = cidx[k][t] % 3;
                        const int yy = e0 + r - 1, xx = f0 + s - 1;
                        const float xv = (yy < 0 || yy >= W || xx < 0 || xx >= W) ? 0.f : x[((size_t)n * C + c) * HW + yy * W + xx];
                        volatile float prod = taps[tb[k] + t].v * xv;
                        o = o + prod;
                    }
                    ++checked;
                    if (o != y[((size_t)n * K + k) * HW + e0 * W + f0]) ++bad;
                }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch_tmr_t<W, KW, WQ, 0>(p, grid, smem, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double macs = (double)N * K * HW * L;
    printf("TMR W=%d KW=%d WQ=%d depth=%d CS=%d NSET=%d smem=%zu enc=%d: %.1f us  %.2f TMAC/s (%.2f of 18.0)  %s/%s/%s  bad %d of %d\n",
           W, KW, WQ, depth, G::CS, G::NSET, smem, (int)cr, ms / reps * 1e3, macs / (ms / reps * 1e-3) / 1e12,
           macs / (ms / reps * 1e-3) / 1e12 / 18.04, cudaGetErrorString(e), cudaGetErrorString(e2),
           cudaGetErrorString(cudaGetLastError()), bad, checked);
#ifdef TMI_TRACE
    static long long tr[2][4096][6];
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
    const int ns = std::min(nst, 4096);
    for (int role = 0; role < 2; ++role) {
        double d[6] = {0};
        for (int s = 1; s < ns; ++s)
            for (int i = 1; i < 6; ++i) d[i] += (double)(tr[role][s][i] - tr[role][s][i - 1]);
        double per = (double)(tr[role][ns - 1][0] - tr[role][1][0]) / (ns - 2);
        printf("  %s: cycles/stage %.0f; segments", role ? "consumer" : "producer", per);
        for (int i = 1; i < 6; ++i) printf(" %.0f", d[i] / (ns - 1));
        printf("\n");
    }
#endif
    cudaFree(dx); cudaFree(dy); cudaFree(dt); cudaFree(dtb); cudaFree(dso);
}

int main(int argc, char** argv) {
    const int reps = 5;
    run_tmr<4, 2, 4>(256, 512, 512, 461, 4, reps);
    run_tmr<4, 2, 4>(256, 512, 512, 461, 4, reps, 0x2000u);  // filler skips the TMEM stores
    run_tmr<4, 2, 4>(256, 512, 512, 461, 4, reps, 0x1000u);  // consumers skip the MACs
    return 0;
}
