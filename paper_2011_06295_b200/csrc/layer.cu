// Device layer objects, the tap-program builder, launch-configuration rules
// and the C-ABI launch entry points.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "variants.h"

using namespace scb;

namespace {

constexpr int kSmemLimit = 227 * 1024 - 1024;  // dynamic limit: 227 KB minus the kernels' static shared memory
constexpr int kMaxThreads = 256;
const int kKtChoices[] = {2, 4, 8};
constexpr int KIND_TILED = 0, KIND_PLANE = 1, KIND_DIRECT = 2, KIND_DIMG = 3, KIND_DWS = 4, KIND_DTM = 5, KIND_TMI = 6,
              KIND_LANE = 7;

// SM count of a device (persistent grids), cached per device
int sm_count(int dev) {
    static int cnt[64];
    if (dev < 0 || dev >= 64) return 148;
    if (cnt[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cnt[dev] = v;
    }
    return cnt[dev];
}

// TMEM image-lane geometry (= tmi.cuh TmiGeom<W, TE, J>)
struct TmiG {
    int W, TE, J, UE, CPR, SROWS, RW, SW, WIN, NSLOT, CS, NSET, IMGS;
    explicit TmiG(const scb_variant_info& v) : W(v.tw), TE(v.th), J(v.nbt) {
        UE = W / TE;
        const bool fullh = TE == W;
        CPR = fullh ? TE + 1 : TE + 2;
        SROWS = fullh ? 3 * CPR + 1 : 3 * CPR;
        RW = J * W;
        SW = SROWS * RW;
        WIN = TE * RW;
        NSLOT = 512 / SW;
        CS = NSLOT >= 8 ? NSLOT / 4 : 1;
        NSET = std::min(8, NSLOT / CS);
        IMGS = 32 * J / UE;
    }
};

scb_status cuda_fail(cudaError_t e, const char* where) {
    return fail(SCB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Tap program of one KT: taps of group g (channels g*KT .. g*KT+KT-1)
// ordered (c, kk, r, s); ptr[g][c] = first tap of channel c in group g.
struct Program {
    int kt = 0;
    int groups = 0;
    std::vector<int32_t> h_ptr;   // groups x (C+1), mask stream
    std::vector<int32_t> h_ptr_j; // groups x (C+1), jump stream
    std::map<int, int> tap_cap;   // cc -> smem tap entries per (stage, group)
    int32_t* d_ptr = nullptr;     // jump stream: ptr[g][c] -> sentinel of first non-empty channel >= c
    Tap* d_taps = nullptr;        // jump stream: per channel a sentinel {KT*R*S, c} + taps; group ends with {., C}
    int32_t* d_ptr_m = nullptr;   // mask stream (taps only)
    Tap* d_taps_m = nullptr;
    uint32_t* d_masks = nullptr;  // groups x C x ceil(KT/2): bit r*S+s of half-word kk
    int64_t ntaps = 0, nentries = 0;
};

}  // namespace

struct scb_layer {
    Geom g{};
    bool has_aq = false;  // activation fake-quant attached (scb_layer_set_act_quant)
    ActQuant aq{};
    scb_dtype dt = SCB_F32;
    scb_wfmt wfmt = SCB_W_NATIVE;
    int wf = WF_F32;
    int device = 0;
    bool unified = true;
    int64_t nnz = 0;
    QuantAux q{};
    // generic-kernel arrays
    void* d_values = nullptr;
    int32_t* d_dec = nullptr;
    int32_t* d_rowptr = nullptr;
    std::vector<Program> progs;
    std::mutex mu;
    // direct-kernel tables, built on first use: taps per (PLANE, ROW) layout, stage pointers per cc
    std::vector<int32_t> h_colidx, h_rowptr;
    std::vector<float> h_vals;     // values as f32 (exact for f16/f32 storage)
    std::vector<uint32_t> h_pay;   // device payload bits (f32 bits, or f16 bits in the low half)
    std::map<std::vector<int>, DirectTap*> d_dtaps;  // key (plane, row, column of each s)
    std::map<int, int32_t*> d_sptr;
    std::map<int, int> sptr_maxseg;  // cc -> longest (channel, stage) tap segment
    std::map<int, std::vector<int32_t>> h_sptr;  // cc -> host copy of the stage pointers
    // stage-major tap blocks of the direct kernel, key (layout..., es, cc, kw):
    // per (channel group g of kw, stage st) one contiguous 16-byte-aligned block
    // [kw int32 counts, padded to 16 B][taps of the kw channels in that stage, kk-major]
    struct Blocks { DirectTap* taps = nullptr; int32_t* off = nullptr; };
    std::map<std::vector<int>, Blocks> d_blocks;
    std::map<std::pair<int, int>, int> blk_cap;  // (cc, kw) -> largest block in 16-byte units
    // TMEM image-lane tables (tmi.cuh), key (SW, CPR, RW, CS): taps {v, TMEM column} per
    // output channel in CSR order, each run padded to an even count (16-byte aligned)
    struct TmiTables { TmiTap* taps = nullptr; int32_t* tbase = nullptr; int32_t* soff = nullptr; int tcap = 0; };
    std::map<std::vector<int>, TmiTables> d_tmi;
    // image-lane position-class tables (lane.cuh), key (cc, nb, u): [st][k][cap] tap slots
    struct LaneTables { uint4* desc = nullptr; uint32_t* zmask = nullptr; int cap = 0; };
    std::map<std::vector<int>, LaneTables> d_lane;
    std::map<std::vector<int>, int> lane_caps;  // host-only slot sizes (launch checks)
    bool finite = true;  // every weight finite: dropping padding taps is exact (lane.cuh)

    // descriptor value words of the lane kernels: f32 bits (f32 kernels, quantized formats
    // decoded), or the f16 kernels' payload (f16 bits / code, decoded in registers)
    std::vector<uint32_t> lane_vbits(int es) const {
        std::vector<uint32_t> vb((size_t)nnz);
        for (int64_t t = 0; t < nnz; ++t) {
            if (es == 2) vb[t] = h_pay[t];
            else std::memcpy(&vb[t], &h_vals[t], 4);
        }
        return vb;
    }
    std::vector<uint8_t> lane_sign() const {
        std::vector<uint8_t> sg((size_t)nnz);
        for (int64_t t = 0; t < nnz; ++t) sg[t] = std::signbit(h_vals[t]) ? 1 : 0;
        return sg;
    }
    bool lane_build(int cc, int nb, int u, int es, bool count_only, LaneProgram* P) const {
        const std::vector<uint32_t> vb = lane_vbits(es);
        const std::vector<uint8_t> sg = lane_sign();
        if (u == 4)  // 4x4 output tiles of any plane with H, W multiples of 4 (lane.cuh k_tile)
            return build_lane_program_tiles(vb.data(), h_colidx.data(), h_rowptr.data(), g.c, g.k,
                                            (int64_t)g.hp * g.wp, g.wp, g.h, g.w, cc, nb, P, count_only, es);
        if (u == 3)  // quadrant tiles of an 8x8 plane (lane.cuh TQ)
            return g.h == 8 && g.w == 8 &&
                   build_lane_program_tq(vb.data(), h_colidx.data(), h_rowptr.data(), g.c, g.k, (int64_t)g.hp * g.wp,
                                         g.wp, cc, nb, P, count_only, es, sg.data());
        return build_lane_program(vb.data(), h_colidx.data(), h_rowptr.data(), g.c, g.k, (int64_t)g.hp * g.wp, g.wp,
                                  g.h, g.w, cc, nb, P, u, count_only, es, sg.data());
    }
    int lane_cap(int cc, int nb, int u, int es) {
        std::lock_guard<std::mutex> lk(mu);
        std::vector<int> key{cc, nb, u, es};
        auto it = lane_caps.find(key);
        if (it != lane_caps.end()) return it->second;
        LaneProgram P;
        const int cap = lane_build(cc, nb, u, es, true, &P) ? P.cap : -1;
        lane_caps[key] = cap;
        return cap;
    }
    LaneTables lane_tables(int cc, int nb, int u, int es, bool build) {
        std::lock_guard<std::mutex> lk(mu);
        std::vector<int> key{cc, nb, u, es};
        auto it = d_lane.find(key);
        if (it != d_lane.end()) return it->second;
        if (!build) return LaneTables{};
        LaneProgram P;
        if (!lane_build(cc, nb, u, es, false, &P)) return LaneTables{};
        LaneTables T;
        T.cap = P.cap;
        if (cudaMalloc(&T.desc, P.desc.size() * 16) != cudaSuccess) return LaneTables{};
        if (cudaMalloc(&T.zmask, P.zmask.size() * 4) != cudaSuccess) { cudaFree(T.desc); return LaneTables{}; }
        if (cudaMemcpy(T.desc, P.desc.data(), P.desc.size() * 16, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(T.zmask, P.zmask.data(), P.zmask.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(T.desc); cudaFree(T.zmask);
            return LaneTables{};
        }
        d_lane[key] = T;
        return T;
    }

    // largest per-channel tap run (even), host only: = tmi_tables().tcap
    int tmi_tcap() const {
        int tcap = 2;
        for (int k = 0; k < g.k; ++k) tcap = std::max(tcap, (h_rowptr[k + 1] - h_rowptr[k] + 1) & ~1);
        return tcap;
    }
    TmiTables tmi_tables(int sw, int cpr, int rw, int cs, int nset, bool build) {
        std::lock_guard<std::mutex> lk(mu);
        std::vector<int> key{sw, cpr, rw, cs, nset};
        auto it = d_tmi.find(key);
        if (it != d_tmi.end()) return it->second;
        if (!build) return TmiTables{};
        const int64_t pp = (int64_t)g.hp * g.wp;
        const int nst = (g.c + cs - 1) / cs;
        std::vector<TmiTap> taps;
        std::vector<int32_t> tb(g.k + 1), so((size_t)g.k * (nst + 1));
        int tcap = 2;
        for (int k = 0; k < g.k; ++k) {
            tb[k] = (int32_t)taps.size();
            int st = 0;
            for (int t = h_rowptr[k]; t < h_rowptr[k + 1]; ++t) {
                const int64_t c = h_colidx[t] / pp, rem = h_colidx[t] % pp;
                const int r = (int)(rem / g.wp), s2 = (int)(rem % g.wp);
                while (st <= nst && (int64_t)st * cs <= c) so[(size_t)k * (nst + 1) + st++] = t - h_rowptr[k];
                TmiTap d;
                const uint32_t vb = native_bits(t);
                std::memcpy(&d.v, &vb, 4);
                d.col = (uint32_t)((c % cs) * sw + (s2 * cpr + r) * rw);
                taps.push_back(d);
            }
            const int cnt = h_rowptr[k + 1] - h_rowptr[k];
            while (st <= nst) so[(size_t)k * (nst + 1) + st++] = cnt;
            if (taps.size() & 1) taps.push_back(TmiTap{0.f, 0u});
            tcap = std::max(tcap, (int)taps.size() - tb[k]);
        }
        tb[g.k] = (int32_t)taps.size();
        TmiTables T;
        T.tcap = tcap;
        if (taps.empty()) taps.push_back(TmiTap{0.f, 0u});
        if (cudaMalloc(&T.taps, taps.size() * sizeof(TmiTap)) != cudaSuccess) return TmiTables{};
        if (cudaMalloc(&T.tbase, tb.size() * 4) != cudaSuccess) { cudaFree(T.taps); return TmiTables{}; }
        if (cudaMalloc(&T.soff, so.size() * 4) != cudaSuccess) { cudaFree(T.taps); cudaFree(T.tbase); return TmiTables{}; }
        if (cudaMemcpy(T.taps, taps.data(), taps.size() * sizeof(TmiTap), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(T.tbase, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(T.soff, so.data(), so.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(T.taps); cudaFree(T.tbase); cudaFree(T.soff);
            return TmiTables{};
        }
        d_tmi[key] = T;
        return T;
    }

    // largest block (16-byte units) for (cc, kw), from the host stage pointers
    // tw = 32-bit words per tap: 2 ({f32 value, byte offset}) or 1 (compact f16 tap)
    int block_cap(int cc, int kw, int tw = 2) {
        host_sptr(cc);
        std::lock_guard<std::mutex> lk(mu);
        auto key = std::make_pair(cc, kw * 4 + tw);
        auto it = blk_cap.find(key);
        if (it != blk_cap.end()) return it->second;
        const std::vector<int32_t>& sp = h_sptr[cc];
        const int nst = (g.c + cc - 1) / cc, groups = (g.k + kw - 1) / kw;
        const int hdr = (kw * 4 + 15) / 16;  // header chunks
        int mx = 1;
        for (int gg = 0; gg < groups; ++gg)
            for (int st = 0; st < nst; ++st) {
                int n = 0;
                for (int kk = 0; kk < kw; ++kk) {
                    const int k = gg * kw + kk;
                    if (k < g.k) n += sp[(size_t)k * (nst + 1) + st + 1] - sp[(size_t)k * (nst + 1) + st];
                }
                mx = std::max(mx, hdr + (n * tw + 3) / 4);
            }
        blk_cap[key] = mx;
        return mx;
    }
    // native value bits of nonzero t (f32 bits, or f16 bits in the low half) whatever the
    // stored weight format: quantized payloads are decoded here, exactly
    uint32_t native_bits(int64_t t) const {
        if (wfmt == SCB_W_NATIVE) return h_pay[t];
        if (dt == SCB_F16) {
            const __half h = __float2half_rn(h_vals[t]);  // exact: the value came from f16
            return (uint32_t)__half_as_ushort(h);
        }
        uint32_t b;
        std::memcpy(&b, &h_vals[t], 4);
        return b;
    }
    // device tables: taps (as 16-byte chunks) and per-(g, st) chunk offsets.  es = 2 (the f16
    // kernels): compact 4-byte taps {element offset relative to the stage (16 bits), payload
    // (16 bits: f16 bits / int16 code / 4-bit codebook index)} decoded in registers
    // (kernels.cuh tap_f16); otherwise 8-byte {native value, byte offset}.
    Blocks direct_blocks(int plane, int row, const std::vector<int>& col, int es, int cc, int kw, bool build) {
        if (build) host_sptr(cc);
        std::lock_guard<std::mutex> lk(mu);
        std::vector<int> key{plane, row, es, cc, kw};
        key.insert(key.end(), col.begin(), col.end());
        auto it = d_blocks.find(key);
        if (it != d_blocks.end()) return it->second;
        if (!build) return Blocks{};
        const bool compact = es == 2;
        const std::vector<int32_t>& sp = h_sptr[cc];
        const int64_t pp = (int64_t)g.hp * g.wp;
        const int nst = (g.c + cc - 1) / cc, groups = (g.k + kw - 1) / kw;
        const int hdr = (kw * 4 + 15) / 16;
        std::vector<uint32_t> out;  // 32-bit words, 4 per 16-byte chunk
        std::vector<int32_t> off((size_t)groups * nst + 1);
        for (int gg = 0; gg < groups; ++gg)
            for (int st = 0; st < nst; ++st) {
                off[(size_t)gg * nst + st] = (int32_t)(out.size() / 4);  // in 16-byte chunks
                const size_t h0 = out.size();
                out.resize(h0 + 4 * hdr, 0u);
                for (int kk = 0; kk < kw; ++kk) {
                    const int k = gg * kw + kk;
                    const int t0 = k < g.k ? sp[(size_t)k * (nst + 1) + st] : 0;
                    const int t1 = k < g.k ? sp[(size_t)k * (nst + 1) + st + 1] : 0;
                    out[h0 + kk] = (uint32_t)(t1 - t0);
                    for (int t = t0; t < t1; ++t) {
                        const int64_t c = h_colidx[t] / pp, rem = h_colidx[t] % pp;
                        if (compact) {
                            const int64_t e = (c - (int64_t)st * cc) * plane + (rem / g.wp) * row + col[rem % g.wp];
                            if (e < 0 || e > 0xffff) return Blocks{};  // (derive rejects such launches)
                            out.push_back((h_pay[t] << 16) | (uint32_t)e);
                        } else {
                            out.push_back(native_bits(t));
                            out.push_back((uint32_t)(int32_t)(es * (c * plane + (rem / g.wp) * row + col[rem % g.wp])));
                        }
                    }
                }
                while (out.size() & 3) out.push_back(0u);
            }
        off[(size_t)groups * nst] = (int32_t)(out.size() / 4);  // end of the last block
        Blocks b;
        const size_t nw = std::max<size_t>(out.size(), 4);
        out.resize(nw, 0u);
        if (cudaMalloc(&b.taps, nw * 4) != cudaSuccess) return Blocks{};
        if (cudaMalloc(&b.off, off.size() * 4) != cudaSuccess) { cudaFree(b.taps); return Blocks{}; }
        if (cudaMemcpy(b.taps, out.data(), nw * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(b.off, off.data(), off.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(b.taps);
            cudaFree(b.off);
            return Blocks{};
        }
        d_blocks[key] = b;
        return b;
    }

    ~scb_layer() {
        DeviceGuard dg(device);
        cudaFree(d_values);
        cudaFree(d_dec);
        cudaFree(d_rowptr);
        for (auto& p : progs) { cudaFree(p.d_ptr); cudaFree(p.d_taps); cudaFree(p.d_ptr_m); cudaFree(p.d_taps_m); cudaFree(p.d_masks); }
        for (auto& kv : d_dtaps) cudaFree(kv.second);
        for (auto& kv : d_sptr) cudaFree(kv.second);
        for (auto& kv : d_blocks) { cudaFree(kv.second.taps); cudaFree(kv.second.off); }
        for (auto& kv : d_tmi) { cudaFree(kv.second.taps); cudaFree(kv.second.tbase); cudaFree(kv.second.soff); }
        for (auto& kv : d_lane) { cudaFree(kv.second.desc); cudaFree(kv.second.zmask); }
    }
    // direct taps {v, c*plane + r*row + s} in CSR order for one shared-memory layout
    DirectTap* direct_taps(int plane, int row, const std::vector<int>& col, int es, bool build) {
        std::lock_guard<std::mutex> lk(mu);
        std::vector<int> key{plane, row, es};
        key.insert(key.end(), col.begin(), col.end());
        auto it = d_dtaps.find(key);
        if (it != d_dtaps.end()) return it->second;
        if (!build) return nullptr;
        const int64_t pp = (int64_t)g.hp * g.wp;
        std::vector<DirectTap> t(nnz + 2);  // +2: bulk copies read up to the next 16-byte boundary
        for (int64_t i = 0; i < nnz; ++i) {
            const int64_t c = h_colidx[i] / pp, rem = h_colidx[i] % pp;
            uint32_t vb = h_pay[i];  // (slack entries stay zero)
            std::memcpy(&t[i].v, &vb, 4);
            t[i].off = (int32_t)(es * (c * plane + (rem / g.wp) * row + col[rem % g.wp]));
        }
        DirectTap* d = nullptr;
        if (cudaMalloc(&d, t.size() * sizeof(DirectTap)) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, t.data(), t.size() * sizeof(DirectTap), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        d_dtaps[key] = d;
        return d;
    }
    // sptr[k][st] = first tap of row k whose input channel is >= st*cc (st = 0..nst), host copy
    // (plus the longest (channel, stage) segment); no device work
    const std::vector<int32_t>& host_sptr(int cc) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = h_sptr.find(cc);
        if (it != h_sptr.end()) return it->second;
        const int64_t pp = (int64_t)g.hp * g.wp;
        const int nst = (g.c + cc - 1) / cc;
        std::vector<int32_t> sp((size_t)g.k * (nst + 1));
        for (int k = 0; k < g.k; ++k) {
            int t = h_rowptr[k];
            for (int st = 0; st <= nst; ++st) {
                const int64_t cmin = (int64_t)st * cc;
                while (t < h_rowptr[k + 1] && h_colidx[t] / pp < cmin) ++t;
                sp[(size_t)k * (nst + 1) + st] = st == nst ? h_rowptr[k + 1] : t;
            }
        }
        int mx = 1;
        for (int k = 0; k < g.k; ++k)
            for (int st = 0; st < nst; ++st)
                mx = std::max(mx, sp[(size_t)k * (nst + 1) + st + 1] - sp[(size_t)k * (nst + 1) + st]);
        sptr_maxseg[cc] = mx;
        return h_sptr[cc] = std::move(sp);
    }
    int maxseg(int cc) {
        host_sptr(cc);
        std::lock_guard<std::mutex> lk(mu);
        return sptr_maxseg[cc];
    }
    // device stage pointers: uploaded by scb_layer_prepare (build), looked up on launch
    int32_t* stage_ptr(int cc, bool build) {
        if (build) host_sptr(cc);
        std::lock_guard<std::mutex> lk(mu);
        auto it = d_sptr.find(cc);
        if (it != d_sptr.end() || !build) return it != d_sptr.end() ? it->second : nullptr;
        const std::vector<int32_t>& sp = h_sptr[cc];
        int32_t* d = nullptr;
        if (cudaMalloc(&d, sp.size() * 4) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        d_sptr[cc] = d;
        return d;
    }
    Program* prog(int kt) {
        for (auto& p : progs) if (p.kt == kt) return &p;
        return nullptr;
    }
    int cap_for(Program& p, int cc) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = p.tap_cap.find(cc);
        if (it != p.tap_cap.end()) return it->second;
        const int C = g.c;
        int mx = 0;
        for (int gg = 0; gg < p.groups; ++gg)
            for (int c0 = 0; c0 < C; c0 += cc) {
                const int c1 = std::min(c0 + cc, C);
                const int a0 = p.h_ptr_j[(size_t)gg * (C + 1) + c0] & ~1;
                const int a1 = p.h_ptr_j[(size_t)gg * (C + 1) + c1] + 2;
                mx = std::max(mx, a1 - a0);
            }
        mx = (mx + 1) & ~1;  // whole 16-byte chunks
        p.tap_cap[cc] = mx;
        return mx;
    }
    const Program* prog(int kt) const {
        for (auto& p : progs) if (p.kt == kt) return &p;
        return nullptr;
    }
};

namespace {

// Derive the device payload of every nonzero for the requested format.
// Returns false (with error set) if the values do not fit the format exactly.
bool encode_payloads(scb_layer* L, const unsigned char* vals, std::vector<uint32_t>& pay,
                     std::vector<float>& as_f32) {
    const int es = dtype_size(L->dt);
    const int64_t nnz = L->nnz;
    pay.resize(nnz);
    as_f32.resize(nnz);
    for (int64_t t = 0; t < nnz; ++t) {
        float f;
        if (L->dt == SCB_F32) std::memcpy(&f, vals + t * es, 4);
        else if (L->dt == SCB_F16) { uint16_t h; std::memcpy(&h, vals + t * 2, 2); __half_raw hr; hr.x = h; f = __half2float(__half(hr)); }
        else { double d; std::memcpy(&d, vals + t * 8, 8); f = (float)d; }
        as_f32[t] = f;
    }
    if (L->wfmt == SCB_W_NATIVE) {
        for (int64_t t = 0; t < nnz; ++t) {
            if (L->dt == SCB_F16) { uint16_t h; std::memcpy(&h, vals + t * 2, 2); pay[t] = h; }
            else { uint32_t b; std::memcpy(&b, &as_f32[t], 4); pay[t] = b; }
        }
        return true;
    }
    if (L->wfmt == SCB_W_CB4) {
        // codebook: the layer's distinct values (bit patterns) form the table
        std::vector<uint32_t> table;
        for (int64_t t = 0; t < nnz; ++t) {
            uint32_t b; std::memcpy(&b, &as_f32[t], 4);
            auto it = std::find(table.begin(), table.end(), b);
            if (it == table.end()) {
                if (table.size() == 16) { set_error("CB4 needs <= 16 distinct weight values"); return false; }
                table.push_back(b);
                it = table.end() - 1;
            }
            pay[t] = (uint32_t)(it - table.begin());
        }
        for (size_t i = 0; i < 16; ++i) {
            uint32_t b = i < table.size() ? table[i] : 0u;
            std::memcpy(&L->q.cb[i], &b, 4);
            L->q.cb16[i] = __half_as_ushort(__float2half_rn(L->q.cb[i]));  // exact for f16 layers
        }
        return true;
    }
    if (L->wfmt == SCB_W_AFF16) {
        // code = round(v / step), accepted iff the storage rounding of f64(code)*step gives v back
        // bit for bit (numpy: dequantize_affine_int in f64, then astype, quantize.py:137-138)
        const double step = L->q.step;
        if (!(step > 0.0) || !std::isfinite(step)) { set_error("AFF16 needs a finite step > 0"); return false; }
        const int es = dtype_size(L->dt);
        for (int64_t t = 0; t < nnz; ++t) {
            const double code0 = std::nearbyint((double)as_f32[t] / step);
            bool ok = false;
            for (int dlt = 0; dlt < 3 && !ok; ++dlt)
                for (int sg : {1, -1}) {
                    const double code = code0 + sg * dlt;
                    if (std::fabs(code) > 32767.0) continue;
                    const double v = 0.0 + code * step;
                    bool same;
                    if (L->dt == SCB_F16) {
                        uint16_t h;
                        std::memcpy(&h, vals + t * es, 2);
                        same = __half_as_ushort(__double2half(v)) == h;
                    } else {
                        uint32_t a, b2;
                        const float fv = (float)v;
                        std::memcpy(&a, &fv, 4);
                        std::memcpy(&b2, vals + t * es, 4);
                        same = a == b2;
                    }
                    if (same) { pay[t] = (uint32_t)(uint16_t)(int16_t)code; ok = true; break; }
                }
            if (!ok) { set_error("AFF16: a value is not the storage rounding of an int16 code x step"); return false; }
        }
        return true;
    }
    // LIN16: v = code * 2^-frac; find the coarsest power-of-two grid holding all values
    int frac = -126;
    for (int64_t t = 0; t < nnz; ++t) {
        float v = as_f32[t];
        if (v == 0.f) continue;
        if (!std::isfinite(v)) { set_error("LIN16 needs finite weights"); return false; }
        int ex;
        float m = std::frexp(v, &ex);  // v = m * 2^ex, |m| in [0.5,1)
        // trailing precision: smallest power of two dividing v
        uint32_t mant = (uint32_t)std::ldexp(std::fabs(m), 24);
        int tz = 0;
        while (tz < 24 && !(mant & (1u << tz))) ++tz;
        int lsb = ex - 24 + tz;  // v is a multiple of 2^lsb
        frac = std::max(frac, -lsb);
    }
    if (frac == -126) frac = 0;
    const float scale = std::ldexp(1.0f, -frac);
    for (int64_t t = 0; t < nnz; ++t) {
        double code = std::ldexp((double)as_f32[t], frac);
        if (std::fabs(code) > 32767.0 || code != std::floor(code)) {
            set_error("LIN16 needs |code| < 2^15 on a common power-of-two grid");
            return false;
        }
        int c = (int)code;
        if ((float)c * scale != as_f32[t]) { set_error("LIN16 decode is not exact"); return false; }
        pay[t] = (uint32_t)(uint16_t)(int16_t)c;
    }
    L->q.scale = scale;
    return true;
}

template <typename T>
scb_status upload(T** dst, const std::vector<T>& v) {
    cudaError_t e = cudaMalloc(dst, std::max<size_t>(v.size(), 1) * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if (!v.empty() && (e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy");
    return SCB_OK;
}

scb_status build_program(scb_layer* L, int kt, const int32_t* colidx, const int32_t* rowptr,
                         const std::vector<uint32_t>& pay) {
    const Geom& g = L->g;
    Program P;
    P.kt = kt;
    P.groups = (g.k + kt - 1) / kt;
    const int C = g.c, RS = g.r * g.s, NW = (kt + 1) / 2;
    const uint32_t sentinel = (uint32_t)(kt * RS);
    const int64_t plane = (int64_t)g.hp * g.wp;
    std::vector<int32_t> ptr_j((size_t)P.groups * (C + 1)), ptr_m((size_t)P.groups * (C + 1));
    std::vector<uint32_t> masks((size_t)P.groups * C * NW, 0u);
    const bool mask_ok = RS <= 16;
    std::vector<Tap> tj, tm, chan;
    tj.reserve(L->nnz + (size_t)P.groups * (C + 1) + 2);
    tm.reserve(L->nnz + 2);
    std::vector<int32_t> cur(kt);
    for (int gg = 0; gg < P.groups; ++gg) {
        for (int kk = 0; kk < kt; ++kk) {
            int k = gg * kt + kk;
            cur[kk] = k < g.k ? rowptr[k] : 0;
        }
        // ptr_j[g][c] must point at the sentinel of the first non-empty channel >= c:
        // fill after the fact, walking channels backwards
        std::vector<int32_t> first_sent(C + 1, -1);
        for (int c = 0; c < C; ++c) {
            ptr_m[(size_t)gg * (C + 1) + c] = (int32_t)tm.size();
            chan.clear();
            for (int kk = 0; kk < kt; ++kk) {
                int k = gg * kt + kk;
                if (k >= g.k) break;
                while (cur[kk] < rowptr[k + 1] && colidx[cur[kk]] / plane == c) {
                    int64_t rem = colidx[cur[kk]] % plane;
                    int r = (int)(rem / g.wp), s = (int)(rem % g.wp);
                    chan.push_back(Tap{(uint32_t)(kk * RS + r * g.s + s), pay[cur[kk]]});
                    if (mask_ok)
                        masks[((size_t)gg * C + c) * NW + kk / 2] |= 1u << (16 * (kk % 2) + r * g.s + s);
                    ++cur[kk];
                }
            }
            if (!chan.empty()) {
                first_sent[c] = (int32_t)tj.size();
                tj.push_back(Tap{sentinel, (uint32_t)c});
                tj.insert(tj.end(), chan.begin(), chan.end());
                tm.insert(tm.end(), chan.begin(), chan.end());
            }
        }
        first_sent[C] = (int32_t)tj.size();
        tj.push_back(Tap{sentinel, (uint32_t)C});  // end-of-group sentinel
        for (int c = C - 1; c >= 0; --c)
            if (first_sent[c] < 0) first_sent[c] = first_sent[c + 1];
        for (int c = 0; c <= C; ++c) ptr_j[(size_t)gg * (C + 1) + c] = first_sent[c];
        ptr_m[(size_t)gg * (C + 1) + C] = (int32_t)tm.size();
    }
    if ((int64_t)tm.size() != L->nnz) return fail(SCB_ERR_FORMAT, "tap program lost entries (colidx order?)");
    for (auto* v : {&tj, &tm}) { v->push_back(Tap{sentinel, 0u}); v->push_back(Tap{sentinel, 0u}); }  // prefetch slack
    P.ntaps = L->nnz;
    P.nentries = (int64_t)tj.size();
    P.h_ptr = ptr_m;
    P.h_ptr_j = ptr_j;
    scb_status st;
    if ((st = upload(&P.d_ptr, ptr_j)) != SCB_OK || (st = upload(&P.d_taps, tj)) != SCB_OK ||
        (st = upload(&P.d_ptr_m, ptr_m)) != SCB_OK || (st = upload(&P.d_taps_m, tm)) != SCB_OK ||
        (st = upload(&P.d_masks, masks)) != SCB_OK) {
        cudaFree(P.d_ptr); cudaFree(P.d_taps); cudaFree(P.d_ptr_m); cudaFree(P.d_taps_m); cudaFree(P.d_masks);
        return st;
    }
    L->progs.push_back(std::move(P));
    return SCB_OK;
}

int wf_of(const scb_layer* L) {
    if (L->wfmt == SCB_W_CB4) return WF_CB4;
    if (L->wfmt == SCB_W_LIN16) return WF_LIN16;
    if (L->wfmt == SCB_W_AFF16) return WF_AFF16;
    return L->dt == SCB_F16 ? WF_F16 : WF_F32;
}

int elem_bytes(const scb_variant_info& v) { return v.io == SCB_F16 ? 2 : 4; }

bool variant_matches(const scb_layer* L, const scb_variant_info& v, uint32_t flags) {
    const Geom& g = L->g;
    if (L->dt == SCB_F64) return false;
    if (g.stride != 1 || v.r != g.r || v.s != g.s || v.pad != g.pad) return false;
    // image-minor activations are the layout of the kind-7 kernels only; an image-minor
    // output from NCHW input is written by the narrow direct kernels, an NCHW output from
    // image-minor input by kind 7
    if (((flags & SCB_FLAG_IMAGE_MINOR) != 0) != (v.kind == KIND_LANE)) return false;
    if ((flags & SCB_FLAG_Y_NCHW) && v.kind != KIND_LANE) return false;
    if ((flags & SCB_FLAG_Y_IMAGE_MINOR) && !(v.kind == KIND_DIRECT && v.dispatch == DISPATCH_JUMP)) return false;
    // f32 direct / image-lane / TMEM kernels take any weight format: their tap blocks carry
    // the decoded native value (decoded once on upload, direct_blocks); the f16 ones decode
    // the compact tap's payload in registers, so their format must match the layer's
    const bool decoded = (v.kind == KIND_DIRECT || v.kind == KIND_DIMG || v.kind == KIND_TMI || v.kind == KIND_LANE) &&
                         L->dt != SCB_F16 && v.wf == WF_F32;
    if (v.io != L->dt || (v.wf != L->wf && !decoded)) return false;
    // f16 storage: FHFMA (exact w.r.t. the reference's f16 profile) always, plus the half2
    // kernels (f16 accumulators) when the caller opts into the fast mode
    const int mode = (L->dt == SCB_F16) ? MODE_FMA : ((flags & SCB_FLAG_FAST) ? MODE_FMA : MODE_EXACT);
    if (v.mode != mode && !(L->dt == SCB_F16 && (flags & SCB_FLAG_FAST) && v.mode == MODE_HALF2)) return false;
    if (v.kind < KIND_DIRECT && !L->prog(v.kt)) return false;
    if (v.kind == KIND_DIMG) {
        if (g.h != v.th || g.w != v.tw || g.r != 3 || g.s != 3 || g.pad != 1) return false;
        return true;
    }
    if (v.kind == KIND_LANE && v.dispatch == 4) {  // 4x4 output tiles: planes of 4-multiples, 8x8 and up
        if (g.h % 4 || g.w % 4 || g.h * g.w < 64 || g.r != 3 || g.s != 3 || g.pad != 1 || !L->finite) return false;
        return true;
    }
    if (v.kind == KIND_LANE) {  // whole H x W plane per lane, 3x3 "same" convolution, finite weights
        if (g.h != v.th || g.w != v.tw || g.r != 3 || g.s != 3 || g.pad != 1 || !L->finite) return false;
        if ((flags & SCB_FLAG_POOL2) && ((g.h & 1) || (g.w & 1))) return false;
        return true;
    }
    if (v.kind == KIND_TMI) {  // square W x W planes, 3x3 "same" convolution
        if (g.h != v.tw || g.w != v.tw || g.r != 3 || g.s != 3 || g.pad != 1) return false;
        if ((flags & SCB_FLAG_POOL2) && (v.th & 1)) return false;
        return true;
    }
    if (v.kind == KIND_DTM) {
        if (g.f != v.tw || (g.w * 4) % 16 != 0 || g.w > 32 || g.r != 3 || g.s != 3 || g.pad != 1) return false;
        if ((flags & SCB_FLAG_POOL2) && ((g.e & 1) || (g.f & 1) || (v.th & 1))) return false;
        return true;
    }
    if (v.kind == KIND_DIRECT && v.dispatch == DISPATCH_ONED)  // 1D rows
        return g.h == 1 && g.e == 1 && !(flags & SCB_FLAG_POOL2);
    if (v.kind == KIND_DIRECT && v.dispatch == DISPATCH_WIDE) {  // column tiles: any row width
        if (v.tw > 8 && g.f <= v.tw / 2) return false;          // a narrower tile fits better
        if (v.tw < 8 && g.f > 2 * v.tw) return false;           // tiny tiles: small planes only
        if ((flags & SCB_FLAG_POOL2) && ((g.e & 1) || (g.f & 1) || (v.th & 1))) return false;
        return true;
    }
    if (v.kind == KIND_DIRECT || v.kind == KIND_DWS) {
        // rows are staged in 16-byte chunks (one chunk when a row is shorter: direct.cuh CB)
        const int cb = v.kind == KIND_DIRECT ? std::min(16, v.tw * elem_bytes(v)) : 16;
        if (g.f != v.tw || (g.w * elem_bytes(v)) % cb != 0 || g.w > 32) return false;
        if ((flags & SCB_FLAG_POOL2) && ((g.e & 1) || (g.f & 1) || (v.th & 1))) return false;
        return true;
    }
    if (v.kind == KIND_PLANE) {
        if (g.h != v.th || g.w != v.tw) return false;
        if ((flags & SCB_FLAG_POOL2) && ((g.e & 1) || (g.f & 1))) return false;
        return true;
    }
    if ((flags & SCB_FLAG_POOL2) && ((v.th & 1) || (v.tw & 1))) return false;
    return true;
}


// smem row pitch (elements) of a zero-halo window row: XOFF (16 bytes) +
// block columns + right halo + one copy chunk of rounding slack, 16-byte rows.
int row_pitch(const scb_variant_info& v, int bw) {
    const int es = elem_bytes(v), q = 16 / es;
    const int need = q + bw + v.s - 1 - v.pad + q;
    return (need + q - 1) / q * q;
}

// Validate a launch and compute its derived quantities.
struct Derived {
    int wp, threads, row, stage_el, chunk, tap_cap, n_ey, n_fx, kblocks, nb;
    size_t smem;
    unsigned grid;
};

// Whole-plane variants (plane.cuh): imgs = wp * 32 * nbt, image pitch
// = (cc*H*W elements rounded up to 128 B) + 16 B.
scb_status derive_plane(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int es = elem_bytes(v);
    const int hw = g.h * g.w;
    if (c.imgs < 32 * v.nbt || c.imgs % (32 * v.nbt) || c.cc < 1 || c.warps_k < 1)
        return fail(SCB_ERR_SHAPE, "plane launch: imgs must be a multiple of 32*nbt");
    if (((int64_t)c.cc * hw * es) % 16 || ((int64_t)g.c * hw * es) % 16)
        return fail(SCB_ERR_SHAPE, "plane launch: channel runs must be 16-byte multiples");
    d->wp = c.imgs / (32 * v.nbt);
    d->threads = c.warps_k * d->wp * 32;
    if (d->threads > kMaxThreads) return fail(SCB_ERR_SHAPE, "too many threads per CTA");
    const size_t run = ((size_t)c.cc * hw * es + 127) & ~(size_t)127;
    d->row = (int)((run + 16) / es);
    const size_t stage_bytes = ((size_t)c.imgs * d->row * es + 127) & ~(size_t)127;
    d->stage_el = (int)(stage_bytes / es);
    d->chunk = 16;
    d->tap_cap = L->cap_for(*L->prog(v.kt), c.cc);
    d->smem = 2 * stage_bytes + (size_t)2 * c.warps_k * d->tap_cap * sizeof(Tap);
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    const Program* P = L->prog(v.kt);
    d->n_ey = 1;
    d->n_fx = 1;
    d->kblocks = (P->groups + c.warps_k - 1) / c.warps_k;
    d->nb = (n + c.imgs - 1) / c.imgs;
    const int64_t grid = (int64_t)d->kblocks * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

// Direct variants (direct.cuh): 32/tw images per CTA, th output rows, warps_k warps.
// = direct.cuh DirectRow<S, PAD, LW = tw, VX = nbt, ES>
int direct_qw(const scb_variant_info& v) {
    const int q = v.io == SCB_F16 ? 8 : 4;  // elements per 16 bytes (= XO)
    const int right = v.s - 1 - v.pad > 0 ? v.s - 1 - v.pad : 0;
    (void)right;  // VX = 1 rows alias the right halo onto the next row's left padding
    if (v.kind == KIND_DIRECT && v.dispatch == DISPATCH_WIDE) return q + v.tw + q;  // real right halo
    if (v.nbt == 1) return (q + v.tw + q - 1) / q * q;
    const int qw = (q + v.tw + v.s + q - 1) / q * q;  // VX = 2: = direct.cuh DirectRow::QW
    return (2 * qw * elem_bytes(v)) % 128 == 0 ? qw + q : qw;
}
int direct_row(const scb_variant_info& v) { return v.nbt * direct_qw(v); }
std::vector<int> direct_cols(const scb_variant_info& v) {
    std::vector<int> col(v.s);
    const int qw = direct_qw(v);
    for (int s = 0; s < v.s; ++s) {
        const int t = s - v.pad;
        const int xo = v.io == SCB_F16 ? 8 : 4;
        col[s] = v.nbt == 1 ? xo - v.pad + s : ((t % 2 == 0) ? xo + t : qw + xo + t + 1);
    }
    return col;
}

// elements per staging copy of a WIDE/ONED direct row (= direct.cuh `ce`): 16, 8 or 4 bytes
int direct_copy_elems(const scb_variant_info& v, int w, int row) {
    const int q = 16 / elem_bytes(v);
    if (v.dispatch != DISPATCH_WIDE && v.dispatch != DISPATCH_ONED)  // = direct.cuh QC
        return std::min(16, v.tw * elem_bytes(v)) / elem_bytes(v);
    if (w % q == 0 && row % q == 0) return q;
    return (w % 2 == 0 && row % 2 == 0) ? 2 : 1;
}

scb_status derive_direct(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int G = 32 * v.nbt / v.tw;
    if (c.imgs != G || c.bh != v.th || c.bw != v.tw || c.cc < 1 || c.warps_k < 1 ||
        32 * c.warps_k > variant(c.variant).max_threads)
        return fail(SCB_ERR_SHAPE, "direct launch: imgs = 32*vx/tw, bh = th, bw = tw, warps within the kernel's bound");
    const int nbuf = c.stages == 0 ? 2 : c.stages;
    if (nbuf < 2 || nbuf > 3) return fail(SCB_ERR_SHAPE, "direct launch: stages must be 2 or 3");
    d->threads = 32 * c.warps_k;
    d->row = direct_row(v);
    const bool oned = v.dispatch == DISPATCH_ONED;
    const int es = elem_bytes(v), q16 = 16 / es;
    const int plane = oned ? q16 + v.th * v.tw + q16 : (v.th + v.r - 1) * d->row;  // = direct.cuh PLANE
    const int ce = direct_copy_elems(v, g.w, d->row);  // image pitch granule (copy alignment)
    int ip = (c.cc * plane + ce - 1) / ce * ce;
    if (G > 1) {  // word pitch of an image = its row width in words (mod 32): conflict-free lanes
        int t = ip;
        for (int i = 0; i < 64 && (t * es / 4) % 32 != (v.tw * es / 4) % 32; ++i) t += ce;
        if ((t * es / 4) % 32 == (v.tw * es / 4) % 32) ip = t;
    }
    d->chunk = ip;  // image pitch (elements) travels in `chunk`
    const size_t stage_bytes = ((size_t)G * ip * es + 16 + 127) & ~(size_t)127;  // +16: zero tail
    d->stage_el = (int)(stage_bytes / es);
    d->tap_cap = plane;  // plane pitch (elements) travels in `tap_cap`
    const int rows = G * c.cc * (oned ? 1 : v.th + v.r - 1);
    const bool compact = v.io == SCB_F16;  // 4-byte taps with 16-bit stage-relative offsets
    if (compact && (int64_t)c.cc * plane > 0x10000) return fail(SCB_ERR_SHAPE, "stage too large for 16-bit tap offsets");
    const int cap = L->block_cap(c.cc, v.kt, compact ? 1 : 2);  // 16-byte chunks per (group, stage) tap block
    d->wp = cap;  // tap block slot (16-byte units) travels in `wp`
    d->smem = nbuf * stage_bytes + (((size_t)rows * 8 + 15) & ~(size_t)15) +
              (size_t)nbuf * c.warps_k * cap * 16;
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    if (2 * stage_bytes >= (1u << 24) * (size_t)es) return fail(SCB_ERR_SHAPE, "stage too large for row descriptors");
    d->n_ey = oned ? 1 : (g.e + v.th - 1) / v.th;
    d->n_fx = v.dispatch == DISPATCH_WIDE ? (g.f + v.tw - 1) / v.tw
              : oned                      ? (g.f + v.th * v.tw - 1) / (v.th * v.tw) : 1;
    d->kblocks = (g.k + c.warps_k * v.kt - 1) / (c.warps_k * v.kt);
    d->nb = (n + G - 1) / G;
    const int64_t grid = (int64_t)d->kblocks * d->n_ey * d->n_fx * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

// Image-lane direct variants (dimg.cuh): 32 images per CTA, (H+2) x 3H floats per (image, channel).
// = dimg.cuh BASE (elements before copy_1's padded row 0 in an (image, channel) block)
int dimg_base(const scb_variant_info& v) {
    return v.io == SCB_F16 ? (v.th == 2 ? 2 : 4) : (v.th == 2 ? 2 : 0);
}

scb_status derive_dimg(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int H = v.th;
    if (c.imgs != 32 || c.bh != H || c.bw != H || c.cc < 1 || c.warps_k < 1 || c.warps_k > 16)
        return fail(SCB_ERR_SHAPE, "image-lane launch: imgs = 32, bh = bw = plane, 1..16 warps");
    const int nbuf = c.stages == 0 ? 2 : c.stages;
    if (nbuf < 2 || nbuf > 3) return fail(SCB_ERR_SHAPE, "image-lane launch: stages must be 2 or 3");
    d->threads = 32 * c.warps_k;
    const int es = elem_bytes(v);
    d->row = H;                             // = dimg.cuh RW / BLK / BASE
    const int blk = (3 * H + 4) * H + (H == 4 ? 32 / elem_bytes(v) : 0);  // = dimg.cuh BLK
    int ip = c.cc * blk + dimg_base(v);
    const int vec = H;                      // elements per vector load
    while ((ip / vec) % 2 == 0 || ip % vec) ++ip;  // odd vector index: conflict-free lanes
    d->chunk = ip;
    const size_t stage_bytes = ((size_t)32 * ip * es + 127) & ~(size_t)127;
    d->stage_el = (int)(stage_bytes / es);
    d->tap_cap = blk;
    const bool compact = v.io == SCB_F16;  // 4-byte taps with 16-bit stage-relative offsets
    if (compact && (int64_t)c.cc * blk > 0x10000) return fail(SCB_ERR_SHAPE, "stage too large for 16-bit tap offsets");
    const int cap = L->block_cap(c.cc, v.kt, compact ? 1 : 2);  // 16-byte chunks per (group, stage) tap block
    d->wp = cap;
    d->smem = nbuf * stage_bytes + (size_t)nbuf * c.warps_k * cap * 16;
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    d->n_ey = 1;
    d->n_fx = 1;
    d->kblocks = (g.k + c.warps_k * v.kt - 1) / (c.warps_k * v.kt);
    d->nb = (n + 31) / 32;
    const int64_t grid = (int64_t)d->kblocks * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

// TMEM-operand direct variants (tm.cuh): 4 lane quarters x nbt warps, 8 channels per stage.
scb_status derive_dtm(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int M = v.nbt, G = 4 * (32 / v.tw), CC = 8;
    if (c.imgs != G || c.bh != v.th || c.bw != v.tw || c.cc != CC || c.warps_k != M)
        return fail(SCB_ERR_SHAPE, "tmem launch: imgs = 4*32/tw, bh = th, bw = tw, cc = 8, warps_k = nbt");
    d->threads = 128 * M;
    scb_variant_info v1 = v;
    v1.nbt = 1;                // nbt means warps per quarter here; the window rows are direct.cuh VX = 1 rows
    d->row = direct_row(v1);
    const int plane = (v.th + v.r - 1) * d->row;
    int ip = (CC * plane + 3) / 4 * 4;
    if (32 / v.tw > 1)
        while (ip % 32 != v.tw % 32) ip += 4;
    d->chunk = ip;
    const size_t stage_bytes = ((size_t)G * ip * 4 + 16 + 127) & ~(size_t)127;
    d->stage_el = (int)(stage_bytes / 4);
    d->tap_cap = 32;  // TMEM columns per channel slot
    const int cap = L->block_cap(CC, v.kt);
    d->wp = cap;
    const int rows = G * CC * (v.th + v.r - 1);
    d->smem = 2 * stage_bytes + (((size_t)rows * 8 + 15) & ~(size_t)15) + (size_t)2 * M * cap * 16;
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    d->n_ey = (g.e + v.th - 1) / v.th;
    d->n_fx = 1;
    d->kblocks = (g.k + M * v.kt - 1) / (M * v.kt);
    d->nb = (n + G - 1) / G;
    const int64_t grid = (int64_t)d->kblocks * d->n_ey * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

// TMEM image-lane variants (tmi.cuh): persistent grid over (lane block, output channel) items.
scb_status derive_tmi(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const TmiG t(v);
    const int WQ = v.dispatch, KW = v.kt;
    const int depth = c.stages == 0 ? 4 : c.stages;
    if (c.warps_k != WQ || c.imgs != t.IMGS || c.bh != t.TE || c.bw != t.W || c.cc != t.CS)
        return fail(SCB_ERR_SHAPE, "tmem image-lane launch: warps_k = WQ, imgs = lane block, bh = TE, bw = W, cc = CS");
    if (depth < 2 || depth > 8) return fail(SCB_ERR_SHAPE, "tmem image-lane launch: stages (filler ring depth) 2..8");
    int ip = (t.CS * g.h * g.w + 3) / 4 * 4;
    while ((ip / 4) % 2 == 0) ip += 4;  // odd 16-byte pitch: a quarter-warp's row loads hit 8 bank groups
    const int stage_fl = (t.IMGS * ip + 31) / 32 * 32;
    const int tcap = L->tmi_tcap();
    const int nst = (g.c + t.CS - 1) / t.CS;
    const int cap = 4 * WQ * KW;
    // four filler rings + the consumers' taps and stage offsets
    d->smem = (size_t)4 * depth * stage_fl * 4 + (size_t)cap * tcap * sizeof(TmiTap) + (size_t)cap * (nst + 1) * 4;
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    d->threads = 32 * (4 + 4 * WQ);
    d->chunk = ip;
    d->stage_el = stage_fl;
    d->tap_cap = tcap;
    d->row = depth;
    d->wp = nst;
    d->n_ey = 1;
    d->n_fx = 1;
    d->nb = (n + t.IMGS - 1) / t.IMGS;
    d->kblocks = 1;
    const int64_t items = (int64_t)d->nb * g.k;
    if (items > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "too many work items");
    d->grid = (unsigned)std::min<int64_t>(items, sm_count(L->device));
    return SCB_OK;
}

// Warp-specialised direct variants (ws.cuh): warps_k consumer warps + 1 producer warp.
scb_status derive_dws(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int G = 32 / v.tw;
    const int nbuf = c.stages == 0 ? 3 : c.stages;
    if (c.imgs != G || c.bh != v.th || c.bw != v.tw || c.cc < 1 || c.warps_k < 1 || c.warps_k > 8 || nbuf < 2 ||
        nbuf > 4)
        return fail(SCB_ERR_SHAPE, "ws launch: imgs = 32/tw, bh = th, bw = tw, 1..8 warps, 2..4 stages");
    d->threads = 32 * (c.warps_k + 1);
    d->row = direct_row(v);
    const int plane = (v.th + v.r - 1) * d->row;
    int ip = (c.cc * plane + 3) / 4 * 4;
    if (G > 1)
        while (ip % 32 != v.tw % 32) ip += 4;
    d->chunk = ip;
    const size_t stage_bytes = ((size_t)G * ip * 4 + 16 + 127) & ~(size_t)127;  // +16: zero tail
    d->stage_el = (int)(stage_bytes / 4);
    d->tap_cap = plane;
    const int segcap = L->maxseg(c.cc);
    d->wp = segcap;
    const int slot = (segcap + 3) & ~1;
    const int np1 = (g.c + c.cc - 1) / c.cc + 1;
    d->smem = nbuf * stage_bytes + (size_t)nbuf * c.warps_k * v.kt * slot * sizeof(DirectTap) +
              (size_t)c.warps_k * v.kt * np1 * 4 + 8 + 2 * nbuf * 8;
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    if ((g.w * 4) % 16) return fail(SCB_ERR_SHAPE, "ws launch: input rows must be 16-byte multiples");
    d->n_ey = (g.e + v.th - 1) / v.th;
    d->n_fx = 1;
    d->kblocks = (g.k + c.warps_k * v.kt - 1) / (c.warps_k * v.kt);
    d->nb = (n + G - 1) / G;
    const int64_t grid = (int64_t)d->kblocks * d->n_ey * d->n_fx * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

// Image-lane position-class variants (lane.cuh): CTA = 32*nb images x warps_k channels,
// + 1 producer warp; stages = ring depth.  d->chunk = slot bytes, d->row = TMA box rows,
// d->tap_cap = descriptor slot units.
scb_status derive_lane(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    const scb_variant_info& v = variant(c.variant).info;
    const Geom& g = L->g;
    const int es = elem_bytes(v);
    const int u = v.dispatch;  // 1 / 2: tap unroll (padded pairs); 3: quadrant tiles (TQ); 4: 4x4 tiles
    const bool tq = u == 3 || u == 4;
    const int HW = u == 4 ? 36 : (tq ? 25 : g.h * g.w), nb = v.nbt, RB = 32 * nb * es;  // staged positions per channel
    const int nbuf = c.stages == 0 ? 2 : c.stages;
    const int maxw = variant(c.variant).max_threads / 32 - 1;
    if (c.imgs != 32 * nb || c.bh != g.h || c.bw != g.w || c.cc < 1 || c.warps_k < 1 || c.warps_k > maxw ||
        nbuf < 2 || nbuf > 4)
        return fail(SCB_ERR_SHAPE, "lane launch: imgs = 32*nb, bh x bw = the plane, warps within the kernel's limit, "
                                   "2..4 stages");
    const int rows = c.cc * HW;
    const int boxrows = tq ? rows : std::min(rows, 256);  // TQ: one 4D box {images, 5, 5, cc}
    if (rows % boxrows || (tq && c.cc > 256))
        return fail(SCB_ERR_SHAPE, "lane launch: cc*H*W must be <= 256 or a multiple of 256");
    const int cap = L->lane_cap(c.cc, nb, u, es);
    if (cap <= 0) return fail(SCB_ERR_SHAPE, "lane launch: tap program does not fit the slot format");
    const int cs = v.kt;  // kind 7: warps per output channel (class split)
    if (c.warps_k % cs) return fail(SCB_ERR_SHAPE, "lane launch: warps must be a multiple of the class split");
    const int kc = c.warps_k / cs;
    const size_t slot = ((size_t)rows * RB + (u == 2 ? (size_t)HW * RB : 0) + (size_t)kc * cap * 16 + 127) & ~(size_t)127;
    d->smem = nbuf * slot + 16 * nbuf;
    // class split + pool: the epilogue exchanges f32 planes through the (drained) ring
    if (cs > 1 && (flags & SCB_FLAG_POOL2))
        d->smem = std::max(d->smem, (size_t)kc * HW * 32 * nb * 4);
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    d->threads = 32 * (c.warps_k + 1);
    d->chunk = (int)slot;
    d->row = boxrows;
    d->tap_cap = cap;
    d->stage_el = nbuf;
    d->kblocks = (g.k + kc - 1) / kc;
    d->nb = (n + 32 * nb - 1) / (32 * nb);
    d->n_ey = d->n_fx = 1;
    d->wp = (g.c + c.cc - 1) / c.cc;
    const int64_t grid = (int64_t)d->kblocks * d->nb * (u == 4 ? (g.h / 4) * (g.w / 4) : (tq ? 4 : 1));
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

scb_status derive(scb_layer* L, const scb_launch& c, int n, uint32_t flags, Derived* d) {
    if (c.variant < 0 || c.variant >= num_variants()) return fail(SCB_ERR_SHAPE, "bad variant index");
    const scb_variant_info& v = variant(c.variant).info;
    if (!variant_matches(L, v, flags)) return fail(SCB_ERR_SHAPE, "variant does not match the layer");
    if (v.kind == KIND_PLANE) return derive_plane(L, c, n, flags, d);
    if (v.kind == KIND_DIRECT) return derive_direct(L, c, n, flags, d);
    if (v.kind == KIND_DIMG) return derive_dimg(L, c, n, flags, d);
    if (v.kind == KIND_DWS) return derive_dws(L, c, n, flags, d);
    if (v.kind == KIND_DTM) return derive_dtm(L, c, n, flags, d);
    if (v.kind == KIND_TMI) return derive_tmi(L, c, n, flags, d);
    if (v.kind == KIND_LANE) return derive_lane(L, c, n, flags, d);
    const Geom& g = L->g;
    const int es = elem_bytes(v);
    if (c.imgs < 1 || c.imgs % v.nbt || c.bh < v.th || c.bh % v.th || c.bw < v.tw || c.bw % v.tw || c.cc < 1 ||
        c.warps_k < 1)
        return fail(SCB_ERR_SHAPE, "launch tile not a multiple of the thread tile");
    const int px = (c.imgs / v.nbt) * (c.bh / v.th) * (c.bw / v.tw);
    if (px % 32) return fail(SCB_ERR_SHAPE, "pixel threads per warp group must be a multiple of 32");
    d->wp = px / 32;
    d->threads = c.warps_k * px;
    if (d->threads > kMaxThreads) return fail(SCB_ERR_SHAPE, "too many threads per CTA");
    if ((flags & SCB_FLAG_POOL2) && ((g.e & 1) || (g.f & 1))) return fail(SCB_ERR_SHAPE, "pool needs even output extents");
    d->row = row_pitch(v, c.bw);
    const size_t plane = (size_t)(c.bh + v.r - 1) * d->row;  // elements per (image, channel)
    const size_t stage_bytes = ((size_t)c.imgs * c.cc * plane * es + 127) & ~(size_t)127;
    d->stage_el = (int)(stage_bytes / es);
    d->tap_cap = 0;
    if (v.dispatch == DISPATCH_JUMP) d->tap_cap = L->cap_for(*L->prog(v.kt), c.cc);
    d->smem = 2 * stage_bytes + (size_t)2 * c.warps_k * d->tap_cap * sizeof(Tap) +
              (size_t)c.imgs * c.cc * (c.bh + v.r - 1) * 8;  // row descriptors
    if (d->smem > (size_t)kSmemLimit) return fail(SCB_ERR_SHAPE, "shared memory over 227 KB");
    if (2 * stage_bytes >= (1u << 24)) return fail(SCB_ERR_SHAPE, "stage too large for row descriptors");
    // copy chunk: the widest of 16/8/4 bytes dividing the input row and the block stride
    const int n_fx = (g.f + c.bw - 1) / c.bw;
    d->chunk = 0;
    for (int ch : {16, 8, 4})
        if (((int64_t)g.w * es) % ch == 0 && (n_fx == 1 || ((int64_t)c.bw * es) % ch == 0)) { d->chunk = ch; break; }
    if (d->chunk == 0) return fail(SCB_ERR_SHAPE, "input rows are not a multiple of 4 bytes");
    if (v.dispatch == DISPATCH_MASK && v.r * v.s > 16) return fail(SCB_ERR_SHAPE, "mask dispatch needs R*S <= 16");
    const Program* P = L->prog(v.kt);
    d->n_ey = (g.e + c.bh - 1) / c.bh;
    d->n_fx = (g.f + c.bw - 1) / c.bw;
    d->kblocks = (P->groups + c.warps_k - 1) / c.warps_k;
    d->nb = (n + c.imgs - 1) / c.imgs;
    const int64_t grid = (int64_t)d->kblocks * d->n_fx * d->n_ey * d->nb;
    if (grid > 0x7fffffffLL) return fail(SCB_ERR_SHAPE, "grid too large");
    d->grid = (unsigned)grid;
    return SCB_OK;
}

int ceil_to(int a, int m) { return (a + m - 1) / m * m; }

// Enumerate launch candidates for a layer and batch.
void enumerate(scb_layer* L, int n, uint32_t flags, std::vector<scb_launch>& out) {
    const Geom& g = L->g;
    const int nv = num_variants();
    for (int vi = 0; vi < nv; ++vi) {
        const scb_variant_info& v = variant(vi).info;
        if (!variant_matches(L, v, flags)) continue;
        if (v.kind == KIND_LANE) {
            for (int wk : {4, 8, 12, 14, 16, 21, 28})
                for (int cc : {4, 8, 12, 16, 24, 32, 48, 64})
                    for (int ns : {2, 3}) {
                        scb_launch c{vi, wk, 32 * v.nbt, g.h, g.w, cc, ns};
                        Derived d;
                        if (derive(L, c, n, flags, &d) == SCB_OK) out.push_back(c);
                    }
            continue;
        }
        if (v.kind == KIND_TMI) {
            const TmiG t(v);
            for (int depth : {3, 5}) {
                scb_launch c{vi, v.dispatch, t.IMGS, t.TE, t.W, t.CS, depth};
                Derived d;
                if (derive(L, c, n, flags, &d) == SCB_OK) out.push_back(c);
            }
            continue;
        }
        if (v.kind == KIND_DTM) {
            scb_launch c{vi, v.nbt, 4 * (32 / v.tw), v.th, v.tw, 8, 2};
            Derived d;
            if (derive(L, c, n, flags, &d) == SCB_OK) out.push_back(c);
            continue;
        }
        if (v.kind == KIND_DWS) {
            for (int wk : {2, 4, 8})
                for (int cc : {4, 8, 16, 32})
                    for (int ns : {3, 4}) {
                        scb_launch c{vi, wk, 32 / v.tw, v.th, v.tw, cc, ns};
                        Derived d;
                        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
                        out.push_back(c);
                    }
            continue;
        }
        if (v.kind == KIND_DIMG) {
            for (int wk : {1, 2, 4, 8, 16})
                for (int cc : {2, 4, 8, 16, 32})
                    for (int ns : {2, 3}) {
                        scb_launch c{vi, wk, 32, v.th, v.tw, cc, ns};
                        Derived d;
                        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
                        out.push_back(c);
                    }
            continue;
        }
        if (v.kind == KIND_DIRECT) {
            for (int wk : {1, 2, 4, 8, 16})
                for (int cc : {4, 8, 16, 32, 64})
                    for (int ns : {2, 3}) {
                        scb_launch c{vi, wk, 32 * v.nbt / v.tw, v.th, v.tw, cc, ns};
                        Derived d;
                        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
                        out.push_back(c);
                    }
            continue;
        }
        if (v.kind == KIND_PLANE) {
            for (int wp : {1, 2, 4}) {
                const int imgs = wp * 32 * v.nbt;
                if (wp > 1 && imgs > ceil_to(n, 32 * v.nbt)) break;
                for (int wk : {1, 2, 4, 8})
                    for (int cc : {4, 8, 16, 32}) {
                        scb_launch c{vi, wk, imgs, g.e, g.f, cc};
                        Derived d;
                        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
                        out.push_back(c);
                    }
            }
            continue;
        }
        std::vector<std::pair<int, int>> blocks;
        const int eh = ceil_to(g.e, v.th), fw = ceil_to(g.f, v.tw);
        blocks.push_back({std::min(eh, 32), std::min(fw, 32)});
        if (eh > 16) blocks.push_back({16, std::min(fw, 32)});
        if (eh > 8 && fw >= 8) blocks.push_back({8, std::min(fw, 32)});
        if (fw > 64) blocks.push_back({std::min(eh, 4), 64});
        for (auto& b : blocks) {
            const int bh = ceil_to(std::min(b.first, eh), v.th), bw = ceil_to(std::min(b.second, fw), v.tw);
            const int tiles = (bh / v.th) * (bw / v.tw);
            int slots = 1;  // smallest image count making the group a whole number of warps
            while ((slots * tiles) % 32) ++slots;
            for (int mult : {1, 2, 4}) {
                const int imgs = slots * mult * v.nbt;
                if (mult > 1 && imgs > ceil_to(n, v.nbt)) break;
                for (int wk : {1, 2, 4, 8}) {
                    for (int cc : {2, 4, 8, 16}) {
                        scb_launch c{vi, wk, imgs, bh, bw, cc};
                        Derived d;
                        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
                        out.push_back(c);
                    }
                }
            }
        }
    }
    set_error("");
}

// Heuristic default (used when the tuner has not run): favour large
// accumulator tiles and enough resident warps, then plane (bulk) staging.
bool pick_default(scb_layer* L, int n, uint32_t flags, int prefer_imgs, scb_launch* out) {
    const Geom& g = L->g;
    std::vector<scb_launch> cands;
    enumerate(L, n, flags, cands);
    if (cands.empty()) return false;
    if (prefer_imgs > 1) {
        std::vector<scb_launch> pref;
        for (auto& c : cands) if (c.imgs == prefer_imgs) pref.push_back(c);
        if (!pref.empty()) cands.swap(pref);
    }
    double best = -1e30;
    for (auto& c : cands) {
        Derived d;
        if (derive(L, c, n, flags, &d) != SCB_OK) continue;
        const scb_variant_info& v = variant(c.variant).info;
        const double warps = (double)d.grid * d.threads / 32.0;
        const double fill = std::min(1.0, warps / (148.0 * 8.0));
        double score;
        if (v.kind >= KIND_DIRECT) {
            // measured on B200 (profiles/r01_probe_*): the dispatch-free kernels win wherever
            // they apply; prefer their tuned shapes -- 8 warps, 16-32 channels per stage,
            // 8 rows x 4-8 channels per warp (direct), 4 channels per warp (image-lane)
            score = 100.0 + 3.0 * std::log(fill + 1e-3);
            if (v.kind == KIND_DWS) score -= 1.0;
            if (c.warps_k == 8) score += 1.0;
            if (v.kind == KIND_DIRECT) {
                // measured (tools/default_vs_tuned.py, profiles/r01_default_vs_tuned.txt): 16-warp
                // CTAs with 32 channels per stage win wherever the input is re-staged for few
                // output-channel work (small planes, 1x1, 1D, wide rows); the dense 32x32 / 16x16
                // layers prefer 8 warps x 16 channels
                const bool few_taps = g.r * g.s <= 3 || g.h * g.w <= 64 || g.f > 32;  // a layer property
                if (c.warps_k == 16) score += few_taps ? 1.3 : 0.8;
                score += few_taps ? (c.cc >= 32 ? 0.8 : 0.0) : (c.cc == 16 ? 0.5 : 0.0);
                score += (v.th == 8 && v.dispatch != DISPATCH_ONED ? 1.0 : 0.0) + (v.kt >= 4 ? 0.5 : 0.0) +
                         (v.nbt == 1 ? 0.3 : 0.0);
                if (v.dispatch == DISPATCH_WIDE && g.f > 32 && fill >= 1.0 && v.tw == 32) score += 0.3;
                if (v.dispatch == DISPATCH_WIDE)  // exact-fit rows first, then the fewest idle lanes
                    score -= 0.4 + 2.0 * (1.0 - (double)g.f / (d.n_fx * v.tw));
                if (v.dispatch == DISPATCH_ONED)  // idle columns of the last tile
                    score -= 3.0 * (1.0 - (double)g.f / (d.n_fx * v.th * v.tw));
            } else if (v.kind == KIND_DIMG) {
                score += (v.kt == 2 ? 0.5 : 0.0) + (c.cc == 32 ? 0.5 : 0.0) + (c.warps_k == 16 ? 1.3 : 0.0) -
                         (g.h == 4 && v.io != SCB_F16 ? 2.0 : 0.0);
            }
            if (v.kind == KIND_LANE) {
                // measured on B200 (tools/lane_harness.cu, profiles/r02_lane_harness_sweep.txt) at
                // batch 256: 4x4 -- 4 images per lane x 3-way class split x 21 warps, cc 12 (111.6 us
                // on conv4_2) or 2 images x 2-way x 28 warps, cc 16 (113.4); 2x2 -- 4 images x 4-way x
                // 28 warps, cc 32 (20.2 us).  Small batches (< 4 image blocks) want one image per lane
                // and the class split (shorter per-warp chains: tools/probe_shard.py).
                const bool small_plane = g.h * g.w <= 4;
                const int blocks = (n + 32 * v.nbt - 1) / (32 * v.nbt);
                score = 200.0 + 3.0 * std::log(fill + 1e-3) + 0.1 * std::log((double)c.cc);
                if (v.dispatch == 3) {  // 8x8 quadrant tiles: conv3_2 139 us at cc 16, 8 warps, 2 slots
                    score += (c.cc == 16 ? 1.0 : 0.0) + (c.warps_k == 8 ? 1.0 : 0.0);
                } else if (v.dispatch == 4 && g.h * g.w <= 64) {  // 4x4 tiles of 8x8: conv3_2 137 us at 1 image
                    score += 2.5 + (v.nbt == 1 ? 1.0 : 0.0) + (c.warps_k == 8 ? 1.0 : 0.0) +  // per lane, 8 warps,
                             (c.cc == 8 ? 1.0 : 0.0) + (c.stages == 2 ? 0.5 : 0.0);          // cc 8, 2 slots
                } else if (v.dispatch == 4) {  // 4x4 tiles: conv2_2 133 us at 2 images / lane, 8 warps, cc 4, 3 slots
                    score += (v.nbt == 2 ? 1.0 : 0.0) + (c.warps_k == 8 ? 1.0 : 0.0) + (c.cc == 4 ? 1.0 : 0.0) +
                             (c.stages == 3 ? 0.5 : 0.0);
                } else if (blocks >= 2) {
                    if (!small_plane && v.nbt == 4 && v.kt == 3 && c.warps_k == 21 && c.cc == 12) score += 2.0;
                    if (!small_plane && v.nbt == 2 && v.kt == 2 && c.warps_k == 28 && c.cc == 16) score += 1.8;
                    if (small_plane && v.nbt == 4 && v.kt == 4 && c.warps_k == 28 && c.cc == 32) score += 2.0;
                } else {
                    score += (v.nbt == 1 ? 1.0 : 0.0) + (v.kt > 1 ? 0.8 : 0.0);
                }
            }
            if (c.stages == 2 || c.stages == 0) score += 0.2;
            // TMEM image-lane kernels: correct, measured slower than direct on VGG-CIFAR
            // (profiles/r02_tmem_*): tuner candidates only, never the untuned default
            if (v.kind == KIND_TMI) score = -100.0;
        } else {
            const double acc = (double)v.kt * v.nbt * v.th * v.tw;  // MACs per tap dispatch
            const double restage = 1.0 / (c.warps_k * v.kt);        // input re-reads per channel
            score = std::log(acc) + 3.0 * std::log(fill + 1e-3) - 2.0 * restage;
            if (c.cc == 8) score += 0.05;
            if (v.kind == KIND_PLANE && g.h * g.w <= 16) {  // 4x4: the measured winner
                score += 50.0 + (v.kt == 2 ? 1.0 : 0.0) + (c.warps_k == 8 ? 1.0 : 0.0) + (c.cc == 16 ? 0.5 : 0.0);
            }
        }
        if (score > best) { best = score; *out = c; }
    }
    set_error("");
    return true;
}

}  // namespace

extern "C" {

SCB_API scb_status scb_layer_create(const scb_shape* shape, scb_dtype dt, scb_wfmt wfmt,
                                    const void* values, const int32_t* colidx,
                                    const int32_t* rowptr, int64_t nnz, int32_t unified,
                                    int32_t device, scb_layer** out) {
    return scb_layer_create_q(shape, dt, wfmt, values, colidx, rowptr, nnz, unified, device, 0.0, out);
}

SCB_API scb_status scb_layer_create_q(const scb_shape* shape, scb_dtype dt, scb_wfmt wfmt,
                                      const void* values, const int32_t* colidx,
                                      const int32_t* rowptr, int64_t nnz, int32_t unified,
                                      int32_t device, double qstep, scb_layer** out) {
    if (!out) return fail(SCB_ERR_ARG, "out is NULL");
    *out = nullptr;
    Geom g;
    scb_status st = make_geom(shape, &g);
    if (st != SCB_OK) return st;
    if (dtype_size(dt) == 0) return fail(SCB_ERR_ARG, "bad dtype");
    if (!rowptr || (nnz > 0 && (!values || !colidx))) return fail(SCB_ERR_ARG, "NULL arrays");
    if (dt == SCB_F64 && wfmt != SCB_W_NATIVE) return fail(SCB_ERR_UNSUPPORTED, "f64 supports native weights only");
    int level = 0;
    for (int k = 0; k < g.k; ++k) level = std::max(level, rowptr[k + 1] - rowptr[k]);
    st = scb_validate_csr(shape, colidx, rowptr, nnz, unified ? 1 : 0, level);
    if (st != SCB_OK) return st;

    DeviceGuard dg(device);
    if (!dg.ok) return fail(SCB_ERR_CUDA, "cannot select device");
    std::unique_ptr<scb_layer> L(new scb_layer());
    L->g = g;
    L->dt = dt;
    L->wfmt = wfmt;
    L->device = device;
    L->unified = unified != 0;
    L->nnz = nnz;
    L->wf = wf_of(L.get());
    L->q.step = qstep;

    std::vector<uint32_t> pay;
    std::vector<float> as_f32;
    if (!encode_payloads(L.get(), static_cast<const unsigned char*>(values), pay, as_f32))
        return SCB_ERR_UNSUPPORTED;

    // generic arrays: native values + decoded (c, r, s)
    const int es = dtype_size(dt);
    const int64_t plane = (int64_t)g.hp * g.wp;
    // decoded taps of the generic kernel: flat kernel index c*R*S + r*S + s (< C*R*S, which
    // scb_validate_csr bounds through colidx < C*Hp*Wp <= 2^31-1)
    std::vector<int32_t> dec(std::max<int64_t>(nnz, 1));
    for (int64_t t = 0; t < nnz; ++t) {
        const int64_t c = colidx[t] / plane, rem = colidx[t] % plane;
        dec[t] = (int32_t)((c * g.r + rem / g.wp) * g.s + rem % g.wp);
    }
    cudaError_t e;
    if ((e = cudaMalloc(&L->d_values, std::max<int64_t>(nnz, 1) * es)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&L->d_dec, dec.size() * 4)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&L->d_rowptr, (g.k + 1) * 4)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if (nnz > 0 && (e = cudaMemcpy(L->d_values, values, nnz * es, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy");
    if ((e = cudaMemcpy(L->d_dec, dec.data(), dec.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy");
    if ((e = cudaMemcpy(L->d_rowptr, rowptr, (g.k + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy");

    L->h_colidx.assign(colidx, colidx + nnz);
    L->h_rowptr.assign(rowptr, rowptr + g.k + 1);
    L->h_vals = as_f32;
    for (float v : as_f32) L->finite &= std::isfinite(v);
    L->h_pay = pay;

    // tiled tap programs for every KT a compiled variant of this (R, S) uses
    if (dt != SCB_F64 && g.stride == 1) {
        for (int kt : kKtChoices) {
            bool used = false;
            for (int vi = 0; vi < num_variants(); ++vi) {
                const auto& v = variant(vi).info;
                used |= (v.kt == kt && v.r == g.r && v.s == g.s && v.io == dt && v.wf == L->wf);
            }
            if (!used) continue;
            st = build_program(L.get(), kt, colidx, rowptr, pay);
            if (st != SCB_OK) return st;
        }
    }
    *out = L.release();
    return SCB_OK;
}

SCB_API scb_status scb_layer_destroy(scb_layer* layer) {
    delete layer;
    return SCB_OK;
}

SCB_API scb_status scb_layer_weight_bytes(const scb_layer* layer, int32_t variant, int64_t* bytes) {
    if (!layer || !bytes) return fail(SCB_ERR_ARG, "NULL");
    auto* L = const_cast<scb_layer*>(layer);
    if (variant < 0) {
        *bytes = L->nnz * (dtype_size(L->dt) + 4) + (int64_t)(L->g.k + 1) * 4;
        return SCB_OK;
    }
    if (variant >= num_variants()) return fail(SCB_ERR_ARG, "bad variant");
    if (scb::variant(variant).info.kind >= KIND_DIRECT) {
        // f16 direct / image-lane kernels: compact 4-byte taps (offset + f16 / code payload)
        const scb_variant_info& vi = scb::variant(variant).info;
        const bool compact = vi.io == SCB_F16 && (vi.kind == KIND_DIRECT || vi.kind == KIND_DIMG);
        *bytes = L->nnz * (compact ? 4 : (int64_t)sizeof(DirectTap)) + (int64_t)(L->g.k + 1) * 4;
        return SCB_OK;
    }
    Program* P = L->prog(scb::variant(variant).info.kt);
    if (!P) return fail(SCB_ERR_ARG, "no program for this variant");
    *bytes = (scb::variant(variant).info.dispatch == DISPATCH_JUMP ? P->nentries : P->ntaps) * (int64_t)sizeof(Tap) +
             (int64_t)P->h_ptr.size() * 4;
    return SCB_OK;
}

SCB_API scb_status scb_launch_candidates(const scb_layer* layer, int32_t n, uint32_t flags,
                                         scb_launch* out, int32_t cap, int32_t* count) {
    if (!layer || !count) return fail(SCB_ERR_ARG, "NULL");
    std::vector<scb_launch> c;
    enumerate(const_cast<scb_layer*>(layer), std::max(n, 1), flags, c);
    *count = (int32_t)c.size();
    for (int i = 0; i < (int)c.size() && i < cap; ++i) out[i] = c[i];
    return SCB_OK;
}

SCB_API scb_status scb_default_launch(const scb_layer* layer, int32_t n, uint32_t flags,
                                      int32_t prefer_imgs, scb_launch* out) {
    if (!layer || !out) return fail(SCB_ERR_ARG, "NULL");
    if ((flags & SCB_FLAG_GENERIC) ||
        !pick_default(const_cast<scb_layer*>(layer), std::max(n, 1), flags, prefer_imgs, out)) {
        *out = scb_launch{-1, 0, 0, 0, 0, 0, 0};
    }
    return SCB_OK;
}

static scb_status conv_sparse_impl(const scb_layer* layer, const void* x, int64_t ldx, const void* bias, void* y,
                                   int64_t ldy, int32_t n, uint32_t flags, const scb_launch* cfg, void* stream,
                                   bool* fused_aq);

// Device tables a launch reads.  build = true (scb_layer_prepare): create and upload them
// (cudaMalloc + synchronous copies).  build = false (scb_conv_sparse): look them up only, so
// the launch path never allocates or synchronises.
struct LaunchTables {
    scb_layer::LaneTables lane;
    const DirectTap* taps = nullptr;
    const int32_t* blkoff = nullptr;
    const int32_t* sptr = nullptr;
    scb_layer::TmiTables tmi;
};
static scb_status launch_tables(scb_layer* L, const scb_launch& c, const Derived& d, bool build, LaunchTables* t) {
    const VariantEntry& ve = variant(c.variant);
    const Geom& g = L->g;
    const char* missing = "launch not prepared: call scb_layer_prepare(layer, n, flags, launch) first";
    if (ve.info.kind == KIND_TMI) {
        const TmiG tg(ve.info);
        t->tmi = L->tmi_tables(tg.SW, tg.CPR, tg.RW, tg.CS, tg.NSET, build);
        if (!t->tmi.taps) return build ? fail(SCB_ERR_CUDA, "tmem image-lane tables: device allocation failed")
                                       : fail(SCB_ERR_ARG, missing);
        return SCB_OK;
    }
    if (ve.info.kind == KIND_LANE) {
        t->lane = L->lane_tables(c.cc, ve.info.nbt, ve.info.dispatch, elem_bytes(ve.info), build);
        if (!t->lane.desc) return build ? fail(SCB_ERR_CUDA, "lane tables: device allocation failed")
                                        : fail(SCB_ERR_ARG, missing);
        return SCB_OK;
    }
    if (ve.info.kind < KIND_DIRECT) return SCB_OK;  // tiled / plane: programs built at layer creation
    std::vector<int> col;
    if (ve.info.kind == KIND_DIMG) {  // = dimg.cuh: BASE + START_s * H, START = {H+1, 0, 2H+2}
        const int H = ve.info.th, start[3] = {H + 1, 0, 2 * H + 2};
        for (int s2 = 0; s2 < g.s; ++s2) col.push_back(dimg_base(ve.info) + start[s2] * H);
    } else {
        col = direct_cols(ve.info);
    }
    if (ve.info.kind == KIND_DTM) {  // tap offsets in TMEM columns: slot(c) + s*RT + r
        col.clear();
        for (int s2 = 0; s2 < g.s; ++s2) col.push_back(s2 * (ve.info.th + g.r - 1));
        auto blk = L->direct_blocks(32, 1, col, 1, c.cc, ve.info.kt, build);
        t->taps = blk.taps;
        t->blkoff = blk.off;
    } else if (ve.info.kind == KIND_DIRECT || ve.info.kind == KIND_DIMG) {
        auto blk = L->direct_blocks(d.tap_cap, d.row, col, elem_bytes(ve.info), c.cc, ve.info.kt, build);
        t->taps = blk.taps;
        t->blkoff = blk.off;
    } else {  // warp-specialised: plain tap array
        t->taps = L->direct_taps(d.tap_cap, d.row, col, elem_bytes(ve.info), build);
        t->blkoff = reinterpret_cast<const int32_t*>(t->taps);  // (unused by ws.cuh; non-null)
    }
    t->sptr = L->stage_ptr(c.cc, build);
    if (!t->taps || !t->blkoff || !t->sptr)
        return build ? fail(SCB_ERR_CUDA, "direct tap tables: device allocation failed") : fail(SCB_ERR_ARG, missing);
    return SCB_OK;
}

SCB_API scb_status scb_layer_prepare(scb_layer* layer, int32_t n, uint32_t flags, const scb_launch* cfg) {
    if (!layer) return fail(SCB_ERR_ARG, "layer is NULL");
    if (n <= 0) return SCB_OK;
    scb_launch c;
    if (cfg) c = *cfg;
    else scb_default_launch(layer, n, flags, 0, &c);
    if (c.variant < 0 || (flags & SCB_FLAG_GENERIC)) return SCB_OK;  // generic: arrays built at creation
    DeviceGuard dg(layer->device);
    if (!dg.ok) return fail(SCB_ERR_CUDA, "cannot select device");
    Derived d;
    scb_status s = derive(layer, c, n, flags, &d);
    if (s != SCB_OK) return s;
    LaunchTables t;
    return launch_tables(layer, c, d, true, &t);
}

SCB_API scb_status scb_launch_check(const scb_layer* layer, int32_t n, uint32_t flags, const scb_launch* cfg) {
    if (!layer || !cfg) return fail(SCB_ERR_ARG, "NULL");
    if (cfg->variant < 0) return SCB_OK;
    Derived d;
    return derive(const_cast<scb_layer*>(layer), *cfg, std::max(n, 1), flags, &d);
}

SCB_API scb_status scb_conv_sparse(const scb_layer* layer, const void* x, const void* bias,
                                   void* y, int32_t n, uint32_t flags,
                                   const scb_launch* cfg, void* stream) {
    return scb_conv_sparse_ld(layer, x, n, bias, y, n, n, flags, cfg, stream);
}

SCB_API scb_status scb_conv_sparse_ld(const scb_layer* layer, const void* x, int64_t ldx, const void* bias, void* y,
                                      int64_t ldy, int32_t n, uint32_t flags, const scb_launch* cfg, void* stream) {
    if (layer && (flags & SCB_FLAG_ACT_QUANT) && !layer->has_aq)
        return fail(SCB_ERR_ARG, "SCB_FLAG_ACT_QUANT on a layer without an activation quantizer");
    bool fused = false;
    scb_status s = conv_sparse_impl(layer, x, ldx, bias, y, ldy, n, flags, cfg, stream, &fused);
    if (s != SCB_OK || !(flags & SCB_FLAG_ACT_QUANT) || fused || n == 0) return s;
    // kernels without the fused epilogue: one in-place pass over the layer output
    const Geom& g = layer->g;
    const bool pool = flags & SCB_FLAG_POOL2;
    const int64_t count = (int64_t)n * g.k * (pool ? g.e / 2 : g.e) * (pool ? g.f / 2 : g.f);
    DeviceGuard dg(layer->device);
    cudaError_t e = launch_fake_quant(layer->dt, y, count, layer->aq, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "fake-quant launch");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

static scb_status conv_sparse_impl(const scb_layer* layer, const void* x, int64_t ldx, const void* bias, void* y,
                                   int64_t ldy, int32_t n, uint32_t flags, const scb_launch* cfg, void* stream,
                                   bool* fused_aq) {
    if (!layer) return fail(SCB_ERR_ARG, "layer is NULL");
    auto* L = const_cast<scb_layer*>(layer);
    if (n < 0) return fail(SCB_ERR_SHAPE, "negative batch");
    if (n == 0) return SCB_OK;
    if (!x || !y) return fail(SCB_ERR_ARG, "NULL activation buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DeviceGuard dg(L->device);
    if (!dg.ok) return fail(SCB_ERR_CUDA, "cannot select device");

    scb_launch c;
    if (cfg) c = *cfg;
    else scb_default_launch(layer, n, flags, 0, &c);
    const Geom& g = L->g;
    // no explicit launch and an input the tiled kernels cannot stage (not 16-byte aligned,
    // e.g. a sliced view): the generic kernel, which accepts any address
    const bool minor = flags & SCB_FLAG_IMAGE_MINOR;
    if (!cfg && (reinterpret_cast<uintptr_t>(x) & 15) && !(flags & SCB_FLAG_POOL2) && !minor) c.variant = -1;
    if (minor && (c.variant < 0 || (flags & SCB_FLAG_GENERIC)))
        return fail(SCB_ERR_UNSUPPORTED, "image-minor activations need a kind-7 (image-lane) launch");
    if (minor && (ldx < n || ldy < n)) return fail(SCB_ERR_ARG, "image-minor row stride smaller than the batch");
    if ((flags & SCB_FLAG_Y_IMAGE_MINOR) && (minor || ldy < n))
        return fail(SCB_ERR_ARG, "SCB_FLAG_Y_IMAGE_MINOR: NCHW input and an output row stride >= the batch");
    if ((flags & SCB_FLAG_Y_NCHW) && !minor) return fail(SCB_ERR_ARG, "SCB_FLAG_Y_NCHW needs SCB_FLAG_IMAGE_MINOR");
    if ((flags & (SCB_FLAG_Y_IMAGE_MINOR | SCB_FLAG_Y_NCHW)) && (c.variant < 0 || (flags & SCB_FLAG_GENERIC)))
        return fail(SCB_ERR_UNSUPPORTED, "output layout flags need a direct / image-lane launch");
    if (c.variant < 0 || (flags & SCB_FLAG_GENERIC)) {
        if (flags & SCB_FLAG_POOL2) return fail(SCB_ERR_UNSUPPORTED, "fused pool needs a tiled variant");
        GenericParams p;
        p.x = x; p.bias = bias; p.y = y; p.values = L->d_values; p.dec = L->d_dec; p.rowptr = L->d_rowptr;
        p.n = n; p.c = g.c; p.h = g.h; p.w = g.w; p.k = g.k; p.e = g.e; p.f = g.f;
        p.stride = g.stride; p.pad = g.pad; p.kr = g.r; p.ks = g.s; p.flags = flags;
        cudaError_t e = launch_generic(p, L->dt, (flags & SCB_FLAG_FAST) != 0, st);
        return e == cudaSuccess ? SCB_OK : cuda_fail(e, "generic kernel launch");
    }
    Derived d;
    scb_status s = derive(L, c, n, flags, &d);
    if (s != SCB_OK) return s;
    const VariantEntry& ve = variant(c.variant);
    if (reinterpret_cast<uintptr_t>(x) & 15) return fail(SCB_ERR_UNSUPPORTED, "tiled kernels need a 16-byte aligned input");
    LaunchTables tab;
    if ((s = launch_tables(L, c, d, false, &tab)) != SCB_OK) return s;
    if (ve.info.kind == KIND_LANE) {
        const int esz = elem_bytes(ve.info);
        if ((ldx * esz) % 16) return fail(SCB_ERR_UNSUPPORTED, "lane kernel: input rows must be 16-byte multiples");
        PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
        if (!enc) return fail(SCB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        LaneParams q;
        std::memset(&q, 0, sizeof(q));
        const int HW = g.h * g.w;
        // quadrant / 4x4 tiles: x as {n, W, H, C}, box {images, 5, 5, cc} / {images, 6, 6, cc}
        const bool tq = ve.info.dispatch == 3 || ve.info.dispatch == 4;
        const cuuint32_t win = ve.info.dispatch == 4 ? 6 : 5;
        const cuuint64_t gdim2[2] = {(cuuint64_t)n, (cuuint64_t)g.c * HW};
        const cuuint64_t gstr2[1] = {(cuuint64_t)ldx * esz};
        const cuuint32_t box2[2] = {(cuuint32_t)(32 * ve.info.nbt), (cuuint32_t)d.row};
        const cuuint64_t gdim4[4] = {(cuuint64_t)n, (cuuint64_t)g.w, (cuuint64_t)g.h, (cuuint64_t)g.c};
        const cuuint64_t gstr4[3] = {(cuuint64_t)ldx * esz, (cuuint64_t)g.w * ldx * esz, (cuuint64_t)HW * ldx * esz};
        const cuuint32_t box4[4] = {(cuuint32_t)(32 * ve.info.nbt), win, win, (cuuint32_t)c.cc};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&q.tmap, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         tq ? 4 : 2, const_cast<void*>(x), tq ? gdim4 : gdim2, tq ? gstr4 : gstr2, tq ? box4 : box2, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SCB_ERR_CUDA, "lane kernel: tensor map encoding failed");
        q.bias = static_cast<const float*>(bias);
        q.y = y;
        q.q = L->q;
        q.desc = tab.lane.desc;
        q.zmask = tab.lane.zmask;
        q.n = n; q.c = g.c; q.k = g.k;
        q.ldx = (int)ldx; q.ldy = (int)ldy;
        q.cc = c.cc; q.nst = d.wp; q.warps = c.warps_k; q.kw = 1;
        q.kgroups = d.kblocks; q.cap = d.tap_cap; q.nbuf = d.stage_el; q.slot_bytes = d.chunk; q.boxrows = d.row;
        q.aq = L->aq;
        q.flags = flags;
        q.h = g.h; q.w = g.w;
        *fused_aq = true;
        if ((int64_t)g.k * (g.e * g.f) * ldy > ((int64_t)1 << 40)) return fail(SCB_ERR_SHAPE, "output too large");
        cudaError_t e = ve.llaunch(q, d.grid, (unsigned)d.threads, d.smem, st);
        return e == cudaSuccess ? SCB_OK : cuda_fail(e, "lane kernel launch");
    }
    if (ve.info.kind == KIND_TMI) {
        const auto& T = tab.tmi;
        TmiParams q;
        std::memset(&q, 0, sizeof(q));
        q.x = static_cast<const float*>(x);
        q.bias = static_cast<const float*>(bias);
        q.y = static_cast<float*>(y);
        q.taps = T.taps; q.tbase = T.tbase; q.soff = T.soff;
        q.n = n; q.c = g.c; q.k = g.k;
        q.nst = d.wp; q.nblk = d.nb; q.depth = d.row; q.ipitch = d.chunk; q.stage_fl = d.stage_el;
        q.tcap = d.tap_cap; q.items = d.nb * g.k;
        q.aq = L->aq;
        q.flags = flags;
        *fused_aq = true;
        if (reinterpret_cast<uintptr_t>(y) & 7) return fail(SCB_ERR_UNSUPPORTED, "tmem image-lane kernel needs an 8-byte aligned output");
        cudaError_t e = ve.tlaunch(q, d.grid, d.smem, st);
        return e == cudaSuccess ? SCB_OK : cuda_fail(e, "tmem image-lane kernel launch");
    }
    if (ve.info.kind >= KIND_DIRECT) {
        DirectParams q;
        std::memset(&q, 0, sizeof(q));
        q.x = x; q.bias = static_cast<const float*>(bias); q.y = y;
        q.taps = tab.taps;
        q.blkoff = tab.blkoff;
        q.sptr = tab.sptr;
        q.n = n; q.c = g.c; q.h = g.h; q.w = g.w; q.k = g.k; q.e = g.e; q.f = g.f;
        q.cc = c.cc; q.nst = (g.c + c.cc - 1) / c.cc; q.wk = c.warps_k;
        q.ip = d.chunk; q.stage_el = d.stage_el;
        q.kblocks = d.kblocks; q.n_ey = d.n_ey; q.nfx = d.n_fx; q.nb = d.nb; q.segcap = d.wp; q.flags = flags;
        q.ldy = ldy;
        q.q = L->q;
        if (ve.info.kind == KIND_DIRECT || ve.info.kind == KIND_DIMG) {  // fused fake-quant epilogue
            q.aq = L->aq;
            *fused_aq = true;
        } else {
            q.flags &= ~SCB_FLAG_ACT_QUANT;
        }
        q.nbuf = c.stages == 0 ? (ve.info.kind == KIND_DWS ? 3 : 2) : c.stages;
        cudaError_t e = ve.dlaunch(q, d.grid, (unsigned)d.threads, d.smem, st);
        return e == cudaSuccess ? SCB_OK : cuda_fail(e, "direct kernel launch");
    }
    const Program* P = L->prog(ve.info.kt);
    TiledParams p;
    std::memset(&p, 0, sizeof(p));
    p.x = x; p.bias = static_cast<const float*>(bias); p.y = y; const bool jump = ve.info.dispatch == DISPATCH_JUMP;
    p.tap_ptr = jump ? P->d_ptr : P->d_ptr_m;
    p.taps = jump ? P->d_taps : P->d_taps_m;
    p.masks = P->d_masks;
    p.q = L->q;
    p.n = n; p.c = g.c; p.h = g.h; p.w = g.w; p.k = g.k; p.e = g.e; p.f = g.f; p.pad = g.pad;
    p.imgs = c.imgs; p.bh = c.bh; p.bw = c.bw; p.cc = c.cc; p.wk = c.warps_k;
    p.wp = d.wp; p.row = d.row; p.stage_el = d.stage_el; p.chunk = d.chunk; p.tap_cap = d.tap_cap;
    p.n_ey = d.n_ey; p.n_fx = d.n_fx; p.kblocks = d.kblocks; p.groups = P->groups;
    p.flags = flags;
    cudaError_t e = ve.launch(p, d.grid, (unsigned)d.threads, d.smem, st);
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "tiled kernel launch");
}

SCB_API scb_status scb_to_image_minor(scb_dtype dt, const void* x, void* y, int32_t n, int64_t chw, int64_t ldy,
                                      void* stream) {
    if (n < 0 || chw < 0 || ldy < n) return fail(SCB_ERR_ARG, "bad extents");
    if (n == 0 || chw == 0) return SCB_OK;
    if (!x || !y) return fail(SCB_ERR_ARG, "NULL buffer");
    cudaError_t e = launch_transpose(dtype_size(dt), x, chw, y, ldy, n, chw, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "transpose launch");
}

SCB_API scb_status scb_from_image_minor(scb_dtype dt, const void* x, int64_t ldx, void* y, int32_t n, int64_t chw,
                                        void* stream) {
    if (n < 0 || chw < 0 || ldx < n) return fail(SCB_ERR_ARG, "bad extents");
    if (n == 0 || chw == 0) return SCB_OK;
    if (!x || !y) return fail(SCB_ERR_ARG, "NULL buffer");
    cudaError_t e = launch_transpose(dtype_size(dt), x, ldx, y, chw, chw, n, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "transpose launch");
}

SCB_API int32_t scb_variant_count(void) { return num_variants(); }

SCB_API scb_status scb_variant_get(int32_t idx, scb_variant_info* out) {
    if (idx < 0 || idx >= num_variants() || !out) return fail(SCB_ERR_ARG, "bad variant index");
    *out = variant(idx).info;
    return SCB_OK;
}

static scb_status make_act_quant(const scb_act_quant* q, scb_dtype dt, ActQuant* out) {
    if (!q) return fail(SCB_ERR_ARG, "act quant is NULL");
    if (q->bits < 1 || q->bits > 31 || !(q->step > 0.0) || (q->symmetric != 0 && q->symmetric != 1))
        return fail(SCB_ERR_ARG, "act quant: bits in 1..31, step > 0, symmetric 0/1");
    ActQuant a{};
    if (dt == SCB_F16) {  // bounds rounded to the activation dtype (numpy's weak python scalars)
        a.lo = __half2float(__double2half(q->clip_lo));
        a.hi = __half2float(__double2half(q->clip_hi));
    } else {
        a.lo = (float)q->clip_lo;
        a.hi = (float)q->clip_hi;
    }
    a.dlo = q->clip_lo;
    a.dhi = q->clip_hi;
    a.mu = q->mu;
    a.step = q->step;
    if (q->symmetric) {
        a.chi = std::ldexp(1.0, q->bits - 1) - 1.0;
        a.clo = -a.chi;
    } else {
        a.clo = 0.0;
        a.chi = std::ldexp(1.0, q->bits) - 1.0;
    }
    *out = a;
    return SCB_OK;
}

SCB_API scb_status scb_layer_set_act_quant(scb_layer* layer, const scb_act_quant* q) {
    if (!layer) return fail(SCB_ERR_ARG, "layer is NULL");
    if (!q) {
        layer->has_aq = false;
        return SCB_OK;
    }
    ActQuant a;
    scb_status s = make_act_quant(q, layer->dt, &a);
    if (s != SCB_OK) return s;
    layer->aq = a;
    layer->has_aq = true;
    return SCB_OK;
}

SCB_API scb_status scb_fake_quant(scb_dtype dt, void* y, int64_t count, const scb_act_quant* q, void* stream) {
    if (count < 0) return fail(SCB_ERR_ARG, "negative count");
    if (count > 0 && !y) return fail(SCB_ERR_ARG, "y is NULL");
    if (dtype_size(dt) == 0) return fail(SCB_ERR_ARG, "bad dtype");
    ActQuant a;
    scb_status s = make_act_quant(q, dt, &a);
    if (s != SCB_OK) return s;
    cudaError_t e = launch_fake_quant(dt, y, count, a, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "fake-quant launch");
}

SCB_API scb_status scb_maxpool2(scb_dtype dt, const void* x, void* y, int64_t planes, int32_t h,
                                int32_t w, void* stream) {
    if ((h & 1) || (w & 1)) return fail(SCB_ERR_SHAPE, "pool needs even extents");
    cudaError_t e = launch_maxpool2(dt, x, y, planes, h, w, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SCB_OK : cuda_fail(e, "maxpool launch");
}

}  // extern "C"
