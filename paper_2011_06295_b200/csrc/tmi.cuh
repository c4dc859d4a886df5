// Tensor-memory image-lane kernel (sm_100a, kind 6): the VGG-CIFAR deep
// layers (W x W planes, W <= 16) with the tap operands in TMEM.
//
// Why: the shared-memory direct kernel (direct.cuh) feeds every exact
// FMUL+FADD pair with one 4-byte shared load; the 128 B/clk/SM shared pipe
// caps it near half the FMUL+FADD rate (profiles/r01_*: 0.27-0.34 in the
// stack).  A tcgen05.ld reads a WARP-UNIFORM column range of each lane's own
// TMEM row at ~256 B/clk/SM (tools/mb_tmem.cu), and the warp-uniform column
// is exactly what an unstructured-sparse tap needs: with every lane holding
// its own input window, one `tcgen05.ld.32x32b.x{WIN}` at column col(c, r, s)
// delivers the WIN operands of tap (c, r, s) for the lane's WIN outputs.  The
// isolated loop runs at 13.3 TMAC/s = 0.74 of the FMUL+FADD peak
// (tools/mb_tmem2.cu) vs 8.0 for the shared-memory loop.
//
// Lane unit = (J images, TE output rows of the full W-wide plane); a lane
// block = 32 units = 32*J/UE images (UE = W/TE row tiles per image).  TMEM
// slot of one input channel, per lane, [copy s][row rho][image j][col phi]:
//   value = xpad[img j][ty*TE + rho - 1][phi + s - 1]      (PAD = 1, R = S = 3)
// so the window of tap (r, s) -- rows r..r+TE-1 of copy s -- is TE*J*W
// CONTIGUOUS columns starting at (s*CPR + r)*J*W.  When a unit covers the
// whole plane height (TE = W) the zero rows of neighbouring copies coincide
// (CPR = TE+1); otherwise CPR = TE+2.  The zero padding (shapes.py:98-105)
// is never read from memory: it is written into TMEM as literal zeros.
//
// CTA = 4 TMEM lane quarters x WQ warps.  All quarters hold the same lane
// block (a TMEM lane quarter is private to the warps w with w % 4 == q), and
// each warp owns KW output channels (compile-time unrolled accumulators).
// Persistent grid: CTA i takes the contiguous range [i*T/G, (i+1)*T/G) of the
// T = blocks*K (lane block, output channel) items, in chunks of at most
// 4*WQ*KW channels of one block.  Input channels stream in stages of CS
// channels: 16-byte cp.async of the block's planes into a D-deep shared ring,
// then each warp copies its share of the stage's channels into two TMEM slot
// sets (shared -> registers -> tcgen05.st), one CTA barrier per stage.
//
// Taps: per output channel the reference CSR row in colidx order
// (csr.py:143-160) as {v, TMEM column}, staged once per chunk in shared
// memory, with per-stage boundaries.  Accumulation per output is bias, then
// v (x) x per tap in colidx order, multiply and add rounded separately in
// exact mode -- bit-identical to _kernels.py:73-84.
#pragma once

#include <cuda_runtime.h>

#include "direct.cuh"
#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

#ifndef TMI_STAMP
#define TMI_STAMP(role, s, i) \
    do {                      \
    } while (0)
#endif

namespace scb {

struct __align__(8) TmiTap {
    float v;
    uint32_t col;  // TMEM column of the tap window relative to its stage set: (c % CS)*SW + window
};

struct TmiParams {
    const float* x;
    const float* bias;      // may be null
    float* y;
    const TmiTap* taps;     // [k] runs at tbase[k] (16-byte aligned), CSR order
    const int32_t* tbase;   // [K+1] first tap of channel k (even)
    const int32_t* soff;    // [K][nst+1] tap index (relative to tbase[k]) of the first tap of stage s
    int n, c, k;
    int nst, nblk;          // stages (CS channels each), lane blocks
    int depth;              // shared input ring depth (stages in flight)
    int ipitch;             // image pitch in the shared stage (floats)
    int stage_fl;           // floats per shared stage
    int tcap;               // taps per warp channel slot in shared memory (even)
    int items;              // nblk * K
    ActQuant aq;
    uint32_t flags;
};

template <int N>
__device__ __forceinline__ void tmi_ld(float (&x)[N], unsigned a);
template <>
__device__ __forceinline__ void tmi_ld<4>(float (&x)[4], unsigned a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void tmi_ld<8>(float (&x)[8], unsigned a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void tmi_ld<16>(float (&x)[16], unsigned a) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15])
        : "r"(a));
}
template <>
__device__ __forceinline__ void tmi_ld<32>(float (&x)[32], unsigned a) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]), "=f"(x[8]),
          "=f"(x[9]), "=f"(x[10]), "=f"(x[11]), "=f"(x[12]), "=f"(x[13]), "=f"(x[14]), "=f"(x[15]), "=f"(x[16]),
          "=f"(x[17]), "=f"(x[18]), "=f"(x[19]), "=f"(x[20]), "=f"(x[21]), "=f"(x[22]), "=f"(x[23]), "=f"(x[24]),
          "=f"(x[25]), "=f"(x[26]), "=f"(x[27]), "=f"(x[28]), "=f"(x[29]), "=f"(x[30]), "=f"(x[31])
        : "r"(a));
}
// register dependency on the loaded window: nothing reads it before the wait
template <int N>
__device__ __forceinline__ void tmi_wait(float (&x)[N]) {
    if constexpr (N == 4) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3])::"memory");
        return;
    }
    static_assert(N == 4 || N % 8 == 0, "window of 4 or 8k columns");
#pragma unroll
    for (int j = 0; j < N; j += 8) {
        if (j == 0)
            asm volatile("tcgen05.wait::ld.sync.aligned;"
                         : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]), "+f"(x[4]), "+f"(x[5]), "+f"(x[6]),
                           "+f"(x[7])::"memory");
        else
            asm volatile(""
                         : "+f"(x[j]), "+f"(x[j + 1]), "+f"(x[j + 2]), "+f"(x[j + 3]), "+f"(x[j + 4]),
                           "+f"(x[j + 5]), "+f"(x[j + 6]), "+f"(x[j + 7]));
    }
}
__device__ __forceinline__ void tmi_st16(unsigned a, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            a),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}

// 16-byte cp.async that allocates in L1: the four lane-quarter fillers of a CTA
// read the same input lines at nearly the same time
__device__ __forceinline__ void cp_async_ca16(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

__device__ __forceinline__ void tmi_st8(unsigned a, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// cp.async.wait_group with a runtime depth (the ring depth is a launch parameter)
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
    switch (n <= 0 ? 0 : (n >= 7 ? 7 : n)) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

// mbarrier primitives (shared::cta)
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
#ifdef MBAR_SPIN
    asm volatile(
        "{\n.reg .pred P;\nWAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n.reg .pred P;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
#endif
}

// Geometry of a variant (host and device agree on it: layer.cu TmiG).
template <int W, int TE, int J>
struct TmiGeom {
    static constexpr int UE = W / TE;                      // row tiles per image
    static constexpr bool FULLH = TE == W;                 // a unit covers the whole plane
    static constexpr int CPR = FULLH ? TE + 1 : TE + 2;    // rows per shifted copy
    static constexpr int SROWS = FULLH ? 3 * CPR + 1 : 3 * CPR;
    static constexpr int RW = J * W;                       // columns per slot row
    static constexpr int SW = SROWS * RW;                  // columns per channel slot
    static constexpr int WIN = TE * RW;                    // window (outputs per lane per channel)
    static constexpr int NSLOT = 512 / SW;
    static constexpr int CS = NSLOT >= 8 ? NSLOT / 4 : 1;  // channels per stage
    static constexpr int NSET = NSLOT / CS > 8 ? 8 : NSLOT / CS;  // TMEM stage sets in the ring
    static constexpr int IMGS = 32 * J / UE;               // images per lane block
    static_assert(W % TE == 0 && 32 % UE == 0, "row tiles");
    static_assert(NSET >= 2, "two channel slots must fit 512 TMEM columns");
    static_assert(SW % 8 == 0, "slots are filled 16 (+8) columns at a time");
};

// Warp roles: warps 0..3 are the FILLERS of TMEM lane quarters 0..3 (global ->
// private cp.async shared ring -> registers -> tcgen05.st); warps 4.. are the
// CONSUMERS (quarter = warp % 4, KW output channels each).  A TMEM stage set
// is handed over with mbarriers (full: filler -> consumers of the quarter,
// empty: consumers -> filler), so no CTA-wide barrier paces the MAC loop and
// the per-stage tap-count imbalance between warps averages out over NSET
// stages of slack.
template <int W, int TE, int J, int KW, int WQ, int MODE>
__global__ void __launch_bounds__(32 * (4 + 4 * WQ), 1) k_tmi(const __grid_constant__ TmiParams p) {
    using G = TmiGeom<W, TE, J>;
    constexpr int UE = G::UE, CPR = G::CPR, RW = G::RW, SW = G::SW, WIN = G::WIN, CS = G::CS, IMGS = G::IMGS;
    constexpr int NSET = G::NSET;
    constexpr int HW = W * W;
    constexpr int NCW = 4 * WQ;         // consumer warps
    constexpr int CAP = NCW * KW;       // output channels per chunk
    constexpr int XR = TE + 2;          // input rows a lane reads per (image, channel)
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned taddr_s;
    __shared__ uint64_t full_b[4][NSET], empty_b[4][NSET];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3;
    const int ig = lane / UE, ty = lane % UE;  // lane unit: image group, row tile
    const int C = p.c, K = p.k;
    const int depth = p.depth;

    // shared: [4 quarters][depth][stage_fl] filler rings | taps [NCW*KW][tcap] | soff [NCW*KW][nst+1]
    float* ring = reinterpret_cast<float*>(smem) + (size_t)q4 * depth * p.stage_fl;
    TmiTap* tsm = reinterpret_cast<TmiTap*>(smem + (size_t)4 * depth * p.stage_fl * 4);
    int32_t* ssm = reinterpret_cast<int32_t*>(tsm + (size_t)CAP * p.tcap);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int q = 0; q < 4; ++q)
            for (int i = 0; i < NSET; ++i) {
                mbar_init(&full_b[q][i], 1);
                mbar_init(&empty_b[q][i], WQ);
            }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tbase = taddr_s + ((unsigned)(32 * q4) << 16);

    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int64_t T = p.items;
    const int64_t a_beg = T * blockIdx.x / gridDim.x, a_end = T * (blockIdx.x + 1) / gridDim.x;
    unsigned g = 0;  // running stage counter (TMEM set = g % NSET, phase = g / NSET)
    for (int64_t a = a_beg; a < a_end;) {
        // equal chunks of at most CAP channels, never crossing a lane block
        const int blk = (int)(a / K);
        const int k0 = (int)(a % K);
        const int64_t left = min(a_end, (int64_t)(blk + 1) * K) - a;
        const int nchunks = (int)((left + CAP - 1) / CAP);
        const int nch = (int)((left + nchunks - 1) / nchunks);
        a += nch;
        const int n0 = blk * IMGS;
        const int nimg = min(IMGS, p.n - n0);

        if (warp < 4) {
            // ================= filler of lane quarter q4 =================
            const float* xg = p.x + (size_t)n0 * C * HW;
            constexpr int RUN4 = CS * HW / 4;  // 16-byte chunks per image of a full stage
            auto load = [&](int s) {
                const int c0 = s * CS;
                const int lim = min(CS, C - c0) * (HW / 4);
                float* dst = ring + (size_t)(s % depth) * p.stage_fl;
                const float* src = xg + (size_t)c0 * HW;
                for (int i = lane; i < nimg * RUN4; i += 32) {
                    const int ib = i / RUN4, q = i - ib * RUN4;
                    if (q < lim) cp_async_ca16(dst + ib * p.ipitch + 4 * q, src + (size_t)ib * C * HW + 4 * q);
                }
            };
            for (int s0 = 0; s0 < depth - 1; ++s0) {
                if (s0 < p.nst) load(s0);
                cp_async_commit();
            }
            for (int s = 0; s < p.nst; ++s, ++g) {
                if (q4 == 0) TMI_STAMP(0, s, 0);
                if (s + depth - 1 < p.nst) load(s + depth - 1);
                cp_async_commit();
                if (q4 == 0) TMI_STAMP(0, s, 1);
                cp_async_wait_dyn(depth - 1);  // this lane's copies of stage s landed
                __syncwarp();                  // ... and every lane's
                if (q4 == 0) TMI_STAMP(0, s, 2);
                const int set = (int)(g % NSET);
                if (g >= NSET) mbar_wait(&empty_b[q4][set], ((g / NSET) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (q4 == 0) TMI_STAMP(0, s, 3);
                const int c0 = s * CS;
                const int ncl = min(CS, C - c0);
                const float* xl = ring + (size_t)(s % depth) * p.stage_fl;
#pragma unroll
                for (int cl = 0; cl < CS; ++cl) {
                    if (cl >= ncl) break;
                    float X[J][XR][W];
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        const int ib = ig * J + j;
                        const bool img_ok = ib < nimg;
                        const float* pl = xl + ib * p.ipitch + cl * HW;
#pragma unroll
                        for (int rho = 0; rho < XR; ++rho) {
                            const int gy = ty * TE + rho - 1;
                            const bool ok = img_ok && gy >= 0 && gy < W;
                            if constexpr (W % 4 == 0) {
#pragma unroll
                                for (int q = 0; q < W / 4; ++q) {
                                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                                    if (ok) v = *reinterpret_cast<const float4*>(pl + gy * W + 4 * q);
                                    X[j][rho][4 * q] = v.x;
                                    X[j][rho][4 * q + 1] = v.y;
                                    X[j][rho][4 * q + 2] = v.z;
                                    X[j][rho][4 * q + 3] = v.w;
                                }
                            } else {
                                static_assert(W == 2, "planes of 2, 4, 8, 16");
                                float2 v = make_float2(0.f, 0.f);
                                if (ok) v = *reinterpret_cast<const float2*>(pl + gy * W);
                                X[j][rho][0] = v.x;
                                X[j][rho][1] = v.y;
                            }
                        }
                    }
                    // slot column -> value: row = s*CPR + rho, (j, phi) inside the row
                    auto sval = [&](int col) -> float {
                        const int row = col / RW, rem = col % RW;
                        const int j = rem / W, phi = rem % W;
                        const int sc = row / CPR, rho = row % CPR;
                        const int gx = phi + sc - 1;
                        return (sc > 2 || gx < 0 || gx >= W) ? 0.f : X[j][rho][gx];
                    };
                    const unsigned sbase = tbase + (unsigned)((set * CS + cl) * SW);
#pragma unroll
                    for (int ch = 0; ch < SW / 16; ++ch) {
                        float v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = sval(ch * 16 + i);
                        tmi_st16(sbase + 16 * ch, v);
                    }
                    if constexpr (SW % 16) {
                        float v[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[i] = sval(SW / 16 * 16 + i);
                        tmi_st8(sbase + SW / 16 * 16, v);
                    }
                }
                if (q4 == 0) TMI_STAMP(0, s, 4);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full_b[q4][set]);
                if (q4 == 0) TMI_STAMP(0, s, 5);
            }
            cp_async_wait<0>();
            continue;
        }

        // ================= consumer: KW output channels =================
        const int cw = warp - 4;
        // taps + stage offsets of this warp's channels -> its own shared slots
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int slot = cw + NCW * kk;
            if (slot < nch) {
                const int k = k0 + slot;
                const int t0 = __ldg(p.tbase + k), t1 = __ldg(p.tbase + k + 1);
                const int4* src = reinterpret_cast<const int4*>(p.taps + t0);
                int4* dst = reinterpret_cast<int4*>(tsm + (size_t)slot * p.tcap);
                for (int i = lane; i < (t1 - t0) / 2; i += 32) cp_async<16>(dst + i, src + i);
                const int32_t* so = p.soff + (size_t)k * (p.nst + 1);
                int32_t* sd = ssm + (size_t)slot * (p.nst + 1);
                for (int i = lane; i <= p.nst; i += 32) sd[i] = __ldg(so + i);
            }
        }
        cp_async_commit();
        float acc[KW][WIN];
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int slot = cw + NCW * kk;
            const float b = (p.bias != nullptr && slot < nch) ? __ldg(p.bias + k0 + slot) : 0.f;
#pragma unroll
            for (int j = 0; j < WIN; ++j) acc[kk][j] = b;
        }
        cp_async_wait<0>();
        __syncwarp();

        for (int s = 0; s < p.nst; ++s, ++g) {
            const int set = (int)(g % NSET);
            if (cw == 0) TMI_STAMP(1, s, 0);
            mbar_wait(&full_b[q4][set], (g / NSET) & 1);
            if (cw == 0) TMI_STAMP(1, s, 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned tset = tbase + (unsigned)(set * CS * SW);
#pragma unroll
            for (int kk = 0; kk < KW; ++kk) {
                const int slot = cw + NCW * kk;
                if (slot >= nch) break;
                const int32_t* so = ssm + (size_t)slot * (p.nst + 1);
                const int t0 = so[s], t1 = so[s + 1];
                const TmiTap* tl = tsm + (size_t)slot * p.tcap;
#pragma unroll 2
                for (int t = t0; t < t1; ++t) {
                    const TmiTap tp = tl[t];
                    float xv[WIN];
                    tmi_ld<WIN>(xv, tset + tp.col);
                    tmi_wait<WIN>(xv);
#pragma unroll
                    for (int j = 0; j < WIN; ++j) acc[kk][j] = mac1<MODE>(acc[kk][j], tp.v, xv[j]);
                }
            }
            if (cw == 0) TMI_STAMP(1, s, 2);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_b[q4][set]);
            if (cw == 0) { TMI_STAMP(1, s, 3); TMI_STAMP(1, s, 4); TMI_STAMP(1, s, 5); }
        }

        // ---- epilogue: window index w = rho_o*RW + j*W + phi -> (n0 + ig*J + j, k, ty*TE + rho_o, phi)
        const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
        const bool relu = p.flags & SCB_FLAG_RELU;
        const bool pool = p.flags & SCB_FLAG_POOL2;
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int slot = cw + NCW * kk;
            if (slot >= nch) break;
            const int k = k0 + slot;
            if (aq) {
#pragma unroll
                for (int j = 0; j < WIN; ++j) acc[kk][j] = fq_store<float>(relu && acc[kk][j] < 0.f ? 0.f : acc[kk][j], p.aq);
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int ib = ig * J + j;
                if (ib >= nimg) continue;
                const int n = n0 + ib;
                if (!pool) {
                    float* yp = p.y + (((int64_t)n * K + k) * W + ty * TE) * W;
#pragma unroll
                    for (int ro = 0; ro < TE; ++ro)
#pragma unroll
                        for (int phi = 0; phi < W; phi += 2) {
                            float o0 = acc[kk][ro * RW + j * W + phi], o1 = acc[kk][ro * RW + j * W + phi + 1];
                            if (relu && !aq) {
                                if (o0 < 0.f) o0 = 0.f;
                                if (o1 < 0.f) o1 = 0.f;
                            }
                            *reinterpret_cast<float2*>(yp + ro * W + phi) = make_float2(o0, o1);
                        }
                } else {
                    constexpr int PW = W / 2;
                    float* yp = p.y + (((int64_t)n * K + k) * PW + ty * (TE / 2)) * PW;
#pragma unroll
                    for (int ro = 0; ro < TE; ro += 2)
#pragma unroll
                        for (int phi = 0; phi < W; phi += 2) {
                            const int b0 = ro * RW + j * W + phi;
                            float o = fmaxf(fmaxf(acc[kk][b0], acc[kk][b0 + 1]),
                                            fmaxf(acc[kk][b0 + RW], acc[kk][b0 + RW + 1]));
                            if (relu && !aq && o < 0.f) o = 0.f;
                            yp[(ro / 2) * PW + phi / 2] = o;
                        }
                }
            }
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int W, int TE, int J, int KW, int WQ, int MODE>
cudaError_t launch_tmi_t(const TmiParams& p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_tmi<W, TE, J, KW, WQ, MODE>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, 32 * (4 + 4 * WQ), smem, st);
}

}  // namespace scb
