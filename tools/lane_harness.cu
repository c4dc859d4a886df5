// Standalone harness for the kind-7 image-lane position-class kernel (csrc/lane.cuh):
// random unified-sparsity 3x3 layer, image-minor activations, bitwise check of a
// sample of images against a CPU loop that runs every tap the reference runs
// (padding taps included, _kernels.py:73-84), then timing of a launch sweep.
//
// build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -Xcompiler -ffp-contract=off -I include -I paper_2011_06295_b200/csrc
//        tools/lane_harness.cu -o tools/lane_harness
// run:   tools/lane_harness H C K L N   (sweeps CS, U, NB, warps, cc, nbuf; 8x8 = quadrant split)
#include <cstdio>
#include <cstdlib>
#include <random>
#include <algorithm>
#include <string>

#include <cudaTypedefs.h>
#include "lane.cuh"

using namespace scb;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

static int g_u = 1, g_cs = 1;
template <int H, int NB, int KW>
cudaError_t launch(const LaneParams& p, unsigned grid, unsigned thr, size_t smem) {
    if (g_cs == 2) {
        if constexpr (H == 8) return cudaErrorInvalidValue;
        else return launch_lane_t<H, H, NB, KW, MODE_EXACT, 1, false, WF_F32, 2>(p, grid, thr, smem, 0);
    }
    if (g_cs == 3) {
        if constexpr (H != 4) return cudaErrorInvalidValue;
        else return launch_lane_t<H, H, NB, KW, MODE_EXACT, 1, false, WF_F32, 3>(p, grid, thr, smem, 0);
    }
    if (g_cs == 4) {
        if constexpr (H == 4) return cudaErrorInvalidValue;
        else return launch_lane_t<H, H, NB, KW, MODE_EXACT, 1, false, WF_F32, 4>(p, grid, thr, smem, 0);
    }
    if (g_u == 2) return launch_lane_t<H, H, NB, KW, MODE_EXACT, 2>(p, grid, thr, smem, 0);
    return launch_lane_t<H, H, NB, KW, MODE_EXACT, 1>(p, grid, thr, smem, 0);
}

static cudaError_t dispatch(int H, int nb, int kw, const LaneParams& p, unsigned grid, unsigned thr, size_t smem) {
#define D(h, b, w) if (H == h && nb == b && kw == w) return launch<h, b, w>(p, grid, thr, smem);
    D(4, 1, 1) D(4, 2, 1) D(4, 4, 1)
    D(2, 2, 1) D(2, 4, 1)
    D(8, 1, 1)
#undef D
    return cudaErrorInvalidValue;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    }
    return fn;
}

// quadrant-tile mode (TQ): 8x8 planes, CTA = (32 images, quadrant, channel group), 5x5 windows
static void run_tq(int C, int K, int L, int N, const std::vector<float>& vals, const std::vector<int32_t>& colidx,
                   const std::vector<int32_t>& rowptr, float* dx, float* dy, float* db, const std::vector<float>& ref,
                   const std::vector<int>& sample) {
    const int HW = 64;
    const double counted = (double)N * K * HW * L;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int cc : {8, 16, 24, 32, 40}) {
        LaneProgram P;
        if (!build_lane_program_tq(reinterpret_cast<const uint32_t*>(vals.data()), colidx.data(), rowptr.data(), C, K, 9,
                                   3, cc, 1, &P))
            continue;
        uint4* dd; uint32_t* dz;
        CK(cudaMalloc(&dd, P.desc.size() * 16));
        CK(cudaMalloc(&dz, P.zmask.size() * 4));
        CK(cudaMemcpy(dd, P.desc.data(), P.desc.size() * 16, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dz, P.zmask.data(), P.zmask.size() * 4, cudaMemcpyHostToDevice));
        for (int wk : {8, 12, 14, 16})
            for (int nbuf : {1, 2, 3}) {
                LaneParams p = {};
                cuuint64_t gdim[4] = {(cuuint64_t)N, 8, 8, (cuuint64_t)C};
                cuuint64_t gstr[3] = {(cuuint64_t)N * 4, (cuuint64_t)N * 32, (cuuint64_t)N * 256};
                cuuint32_t box[4] = {32, 5, 5, (cuuint32_t)cc};
                cuuint32_t es[4] = {1, 1, 1, 1};
                if (encode_fn()(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, gdim, gstr, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                    continue;
                p.boxrows = cc * 25;
                p.bias = db; p.y = dy; p.desc = dd; p.zmask = dz;
                p.n = N; p.c = C; p.k = K; p.ldx = N; p.ldy = N;
                p.cc = cc; p.nst = (C + cc - 1) / cc; p.warps = wk; p.kw = 1;
                p.kgroups = (K + wk - 1) / wk;
                p.cap = P.cap; p.nbuf = nbuf;
                p.slot_bytes = ((cc * 25 * 128 + wk * P.cap * 16) + 127) & ~127;
                const size_t smem = (size_t)nbuf * p.slot_bytes + 16 * nbuf;
                if (smem > 227 * 1024) continue;
                const unsigned grid = (unsigned)(((N + 31) / 32) * 4 * p.kgroups);
                auto go = [&]() { return launch_lane_t<8, 8, 1, 1, MODE_EXACT, 1, false, WF_F32, 1, 1>(p, grid, 32 * (wk + 1), smem, 0); };
                CK(cudaMemset(dy, 0xff, (size_t)K * HW * N * 4));
                cudaError_t e = go();
                if (e != cudaSuccess) { printf("tq cc %d wk %d nbuf %d: %s\n", cc, wk, nbuf, cudaGetErrorString(e)); cudaGetLastError(); continue; }
                CK(cudaDeviceSynchronize());
                std::vector<float> y((size_t)K * HW * N);
                CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
                size_t bad = 0;
                for (size_t si = 0; si < sample.size(); ++si)
                    for (int q = 0; q < K * HW; ++q) {
                        const float a = y[(size_t)q * N + sample[si]], b = ref[(size_t)q * sample.size() + si];
                        if (memcmp(&a, &b, 4) != 0) ++bad;
                    }
                for (int i = 0; i < 3; ++i) go();
                CK(cudaEventRecord(e0));
                for (int i = 0; i < 20; ++i) go();
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const double us = ms * 1000.0 / 20;
                printf("tq cc %2d wk %2d nbuf %d grid %4u smem %6zu: %8.2f us  counted %5.2f TMAC/s  %s\n", cc, wk, nbuf,
                       grid, smem, us, counted / us * 1e-6, bad ? "MISMATCH" : "bitwise");
            }
        cudaFree(dd); cudaFree(dz);
    }
}

int main(int argc, char** argv) {
    const int H = argc > 1 ? atoi(argv[1]) : 4;
    const int C = argc > 2 ? atoi(argv[2]) : 512;
    const int K = argc > 3 ? atoi(argv[3]) : 512;
    const int L = argc > 4 ? atoi(argv[4]) : 461;
    const int N = argc > 5 ? atoi(argv[5]) : 256;
    const int HW = H * H;
    std::mt19937 rng(1234);
    std::normal_distribution<float> nd(0.f, 1.f);
    // unified CSR: L distinct (c, r, s) per channel, colidx order
    std::vector<int32_t> colidx((size_t)K * L), rowptr(K + 1);
    std::vector<float> vals((size_t)K * L), bias(K);
    std::vector<int> perm(C * 9);
    for (int i = 0; i < C * 9; ++i) perm[i] = i;
    for (int k = 0; k < K; ++k) {
        std::shuffle(perm.begin(), perm.end(), rng);
        std::sort(perm.begin(), perm.begin() + L);
        for (int t = 0; t < L; ++t) {
            colidx[(size_t)k * L + t] = perm[t];
            vals[(size_t)k * L + t] = nd(rng) * 0.05f;
        }
        rowptr[k] = k * L;
        bias[k] = nd(rng);
    }
    rowptr[K] = K * L;
    std::vector<float> x((size_t)C * HW * N);
    for (auto& v : x) v = std::max(0.f, nd(rng));
    // CPU reference on a sample of images (all taps, padding included)
    std::vector<int> sample;
    for (int n = 0; n < std::min(N, 40); ++n) sample.push_back(n);
    for (int n = std::max(40, N - 24); n < N; ++n) sample.push_back(n);
    std::vector<float> ref((size_t)K * HW * sample.size());
    for (size_t si = 0; si < sample.size(); ++si) {
        const int n = sample[si];
        for (int k = 0; k < K; ++k)
            for (int yy = 0; yy < H; ++yy)
                for (int xx = 0; xx < H; ++xx) {
                    float o = bias[k];
                    for (int t = rowptr[k]; t < rowptr[k + 1]; ++t) {
                        const int c = colidx[t] / 9, r = colidx[t] / 3 % 3, s = colidx[t] % 3;
                        const int iy = yy + r - 1, ix = xx + s - 1;
                        const float xv = (iy < 0 || iy >= H || ix < 0 || ix >= H) ? 0.f : x[((size_t)c * HW + iy * H + ix) * N + n];
                        const float pr = vals[t] * xv;
                        o = o + pr;
                    }
                    ref[((size_t)k * HW + yy * H + xx) * sample.size() + si] = o;
                }
    }
    float *dx, *dy, *db;
    CK(cudaMalloc(&dx, x.size() * 4));
    CK(cudaMalloc(&dy, (size_t)K * HW * N * 4));
    CK(cudaMalloc(&db, K * 4));
    CK(cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, bias.data(), K * 4, cudaMemcpyHostToDevice));
    if (H == 8 && argc > 6 && std::string(argv[6]) == "tq") {
        run_tq(C, K, L, N, vals, colidx, rowptr, dx, dy, db, ref, sample);
        return 0;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double counted = (double)N * K * HW * L;
    printf("layer H=W=%d C=%d K=%d L=%d N=%d  counted MACs %.3e  SMs %d\n", H, C, K, L, N, counted, sms);
    const int nbs[] = {2, 4}, kws[] = {1}, wks[] = {21, 28}, ccs[] = {8, 12, 16}, nbufs[] = {2, 3}, us[] = {1};
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 1e30;
    // optional single config: argv[6..10] = nb kw wk cc nbuf
    const bool one = argc > 11;
    for (int cs : {2, 3}) for (int u : us) for (int nb : nbs) for (int kw : kws) for (int cc : ccs) {
        g_cs = cs;
        if (one && (nb != atoi(argv[6]) || kw != atoi(argv[7]) || cc != atoi(argv[9]) || u != atoi(argv[11]))) continue;
        if (H != 4 || (cs == 2 && nb == 4)) continue;
        g_u = u;
        LaneProgram P;
        if (!build_lane_program(reinterpret_cast<const uint32_t*>(vals.data()), colidx.data(), rowptr.data(), C, K, 9, 3, H, H,
                                cc, nb, &P, u)) continue;
        uint4* dd; uint32_t* dz;
        CK(cudaMalloc(&dd, P.desc.size() * 16));
        CK(cudaMalloc(&dz, P.zmask.size() * 4));
        CK(cudaMemcpy(dd, P.desc.data(), P.desc.size() * 16, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dz, P.zmask.data(), P.zmask.size() * 4, cudaMemcpyHostToDevice));
        for (int wk : wks) for (int nbuf : nbufs) {
            if (one && (wk != atoi(argv[8]) || nbuf != atoi(argv[10]))) continue;
            LaneParams p = {};
            const int boxrows = std::min(cc * HW, 256);
            if (cc * HW > 1024) continue;
            if ((cc * HW) % boxrows) continue;
            {
                cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)C * HW};
                cuuint64_t gstr[1] = {(cuuint64_t)N * 4};
                cuuint32_t box[2] = {(cuuint32_t)(32 * nb), (cuuint32_t)boxrows};
                cuuint32_t es[2] = {1, 1};
                CUresult r = encode_fn()(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, gdim, gstr, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
            }
            p.boxrows = boxrows;
            p.bias = db; p.y = dy; p.desc = dd; p.zmask = dz;
            p.n = N; p.c = C; p.k = K; p.ldx = N; p.ldy = N;
            p.cc = cc; p.nst = (C + cc - 1) / cc; p.warps = wk; p.kw = kw;
            if (wk % cs || (cs == 1 && wk > 16)) continue;
            const int KC = wk / cs * kw;
            p.kgroups = (K + KC - 1) / KC;
            p.cap = P.cap; p.nbuf = nbuf;
            p.slot_bytes = ((cc * HW * 128 * nb * (u > 1 ? 1 : 1) + (u > 1 ? HW * 128 * nb : 0) + KC * P.cap * 16) + 127) & ~127;
            p.flags = 0;
            const size_t smem = (size_t)nbuf * p.slot_bytes + 16 * nbuf;
            if (smem > 227 * 1024) continue;
            const unsigned grid = (unsigned)(((N + 32 * nb - 1) / (32 * nb)) * p.kgroups);
            CK(cudaMemset(dy, 0xff, (size_t)K * HW * N * 4));
            cudaError_t e = dispatch(H, nb, kw, p, grid, 32 * (wk + 1), smem);
            if (e != cudaSuccess) { printf("nb %d kw %d wk %d cc %d nbuf %d: launch %s\n", nb, kw, wk, cc, nbuf, cudaGetErrorString(e)); cudaGetLastError(); continue; }
            CK(cudaDeviceSynchronize());
            std::vector<float> y((size_t)K * HW * N);
            CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
            size_t bad = 0;
            for (size_t si = 0; si < sample.size(); ++si)
                for (int q = 0; q < K * HW; ++q) {
                    const float a = y[(size_t)q * N + sample[si]], b = ref[(size_t)q * sample.size() + si];
                    if (memcmp(&a, &b, 4) != 0) {
                        if (bad < 3) printf("  mismatch n=%d q=%d gpu %.9g ref %.9g\n", sample[si], q, a, b);
                        ++bad;
                    }
                }
            for (int i = 0; i < 3; ++i) dispatch(H, nb, kw, p, grid, 32 * (wk + 1), smem);
            const int reps = 20;
            CK(cudaEventRecord(e0));
            for (int i = 0; i < reps; ++i) dispatch(H, nb, kw, p, grid, 32 * (wk + 1), smem);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double us = ms * 1000.0 / reps;
            best = std::min(best, us);
            printf("cs %d u %d nb %d kw %d wk %2d cc %2d nbuf %d grid %4u smem %6zu: %8.2f us  counted %5.2f TMAC/s  executed %5.2f TMAC/s  %s\n",
                   cs, u, nb, kw, wk, cc, nbuf, grid, smem, us, counted / us * 1e-6, (double)P.macs * N / us * 1e-6,
                   bad ? "MISMATCH" : "bitwise");
        }
        cudaFree(dd); cudaFree(dz);
    }
    printf("best %.2f us\n", best);
    return 0;
}
