// Host-side unified-sparsity CSR builder, bit-exact with the reference
// build_csr / select_padding_zeros / analyze_sparsity / validate / decompress
// (csr.py:33-178, paths relative to /root/reference/pkg/src/sparseconv).
//
// Works on raw element bytes so the promoted-zero sign bit survives exactly as
// in the numpy gather at csr.py:156.  Zero promotion (csr.py:94-117):
//   key(zero j) = (distance to the nearest ORIGINAL nonzero, j); take the
//   `deficit` smallest keys, emit them ascending; a channel without nonzeros
//   takes its lowest-index zeros.
// Implemented as two linear sweeps for the distances and a counting sort over
// distance buckets (stable in j), O(vol) per channel.
#include <algorithm>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"

namespace scb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

scb_status fail(scb_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

scb_status make_geom(const scb_shape* sh, Geom* g) {
    if (!sh) return fail(SCB_ERR_ARG, "shape is NULL");
    g->n = sh->n; g->c = sh->c; g->h = sh->h; g->w = sh->w; g->k = sh->k;
    g->r = sh->r; g->s = sh->s; g->stride = sh->stride; g->pad = sh->padding;
    if (g->c < 1 || g->h < 1 || g->w < 1 || g->k < 1 || g->r < 1 || g->s < 1 || g->stride < 1)
        return fail(SCB_ERR_SHAPE, "all extents and the stride must be >= 1");
    if (g->pad < 0) return fail(SCB_ERR_SHAPE, "padding must be >= 0");
    g->hp = g->h + 2 * g->pad;
    g->wp = g->w + 2 * g->pad;
    if (g->r > g->hp || g->s > g->wp) return fail(SCB_ERR_SHAPE, "kernel larger than padded input");
    if ((g->hp - g->r) % g->stride || (g->wp - g->s) % g->stride)
        return fail(SCB_ERR_SHAPE, "(extent + 2*padding - kernel) not divisible by stride");
    g->e = (g->hp - g->r) / g->stride + 1;
    g->f = (g->wp - g->s) / g->stride + 1;
    return SCB_OK;
}

// Zero promotion for one flat channel; appends chosen indices (ascending).
static bool promote_zeros(const unsigned char* row, int es, int64_t len, int64_t deficit,
                          std::vector<int64_t>& chosen) {
    chosen.clear();
    if (deficit <= 0) return true;
    std::vector<int64_t> dist(len);
    const int64_t INF = std::numeric_limits<int64_t>::max();
    int64_t nzeros = 0;
    int64_t prev = -1;
    for (int64_t j = 0; j < len; ++j) {
        if (!elem_is_zero(row + j * es, es)) { prev = j; dist[j] = -1; continue; }
        ++nzeros;
        dist[j] = prev < 0 ? INF : j - prev;
    }
    if (deficit > nzeros) return false;
    int64_t next = -1;
    for (int64_t j = len - 1; j >= 0; --j) {
        if (dist[j] < 0) { next = j; continue; }
        if (next >= 0) dist[j] = std::min(dist[j], next - j);
    }
    // counting sort by distance; distances are in [1, len) or INF (no nonzero
    // at all, where index order alone decides -- csr.py:105-106)
    std::vector<int64_t> bucket_count(len + 1, 0);
    for (int64_t j = 0; j < len; ++j)
        if (dist[j] >= 0) ++bucket_count[dist[j] == INF ? len : dist[j]];
    // find the distance threshold holding the deficit-th key
    int64_t take_all_below = 0, acc = 0;
    for (; take_all_below <= len; ++take_all_below) {
        if (acc + bucket_count[take_all_below] >= deficit) break;
        acc += bucket_count[take_all_below];
    }
    int64_t room_at_threshold = deficit - acc;  // lowest-index zeros of that bucket
    for (int64_t j = 0; j < len; ++j) {
        if (dist[j] < 0) continue;
        int64_t b = dist[j] == INF ? len : dist[j];
        if (b < take_all_below) chosen.push_back(j);
        else if (b == take_all_below && room_at_threshold > 0) { chosen.push_back(j); --room_at_threshold; }
    }
    return true;  // already ascending in j
}

}  // namespace scb

using namespace scb;

extern "C" {

SCB_API scb_status scb_channel_nnz(const void* w, scb_dtype dt, int32_t k, int64_t vol,
                                   int64_t* nnz_out) {
    int es = dtype_size(dt);
    if (!w || !nnz_out || es == 0 || k < 0 || vol < 0) return fail(SCB_ERR_ARG, "bad arguments");
    const unsigned char* b = static_cast<const unsigned char*>(w);
    for (int32_t ch = 0; ch < k; ++ch) {
        int64_t cnt = 0;
        const unsigned char* row = b + (int64_t)ch * vol * es;
        for (int64_t j = 0; j < vol; ++j) cnt += !elem_is_zero(row + j * es, es);
        nnz_out[ch] = cnt;
    }
    return SCB_OK;
}

SCB_API scb_status scb_select_padding_zeros(const void* flat, scb_dtype dt, int64_t len,
                                            int64_t deficit, int64_t* out) {
    int es = dtype_size(dt);
    if (es == 0 || len < 0 || deficit < 0) return fail(SCB_ERR_ARG, "bad arguments");
    if (deficit == 0) return SCB_OK;
    if (!flat || !out) return fail(SCB_ERR_ARG, "NULL buffer");
    std::vector<int64_t> chosen;
    if (!promote_zeros(static_cast<const unsigned char*>(flat), es, len, deficit, chosen))
        return fail(SCB_ERR_SHAPE, "deficit " + std::to_string(deficit) + " exceeds available zeros");
    std::copy(chosen.begin(), chosen.end(), out);
    return SCB_OK;
}

SCB_API scb_status scb_csr_count(const void* w, scb_dtype dt, const scb_shape* shape,
                                 int32_t unify, int64_t* nnz_out, int32_t* level_out) {
    Geom g;
    scb_status st = make_geom(shape, &g);
    if (st != SCB_OK) return st;
    int es = dtype_size(dt);
    if (!w || es == 0) return fail(SCB_ERR_ARG, "bad weights");
    if ((int64_t)g.c * g.hp * g.wp > 2147483647LL)
        return fail(SCB_ERR_SHAPE, "padded input volume exceeds 32-bit offset range");
    int64_t vol = (int64_t)g.c * g.r * g.s;
    std::vector<int64_t> cnt(g.k);
    scb_channel_nnz(w, dt, g.k, vol, cnt.data());
    int64_t mx = 0, total = 0;
    for (int64_t v : cnt) { mx = std::max(mx, v); total += v; }
    if (nnz_out) *nnz_out = unify ? mx * g.k : total;
    if (level_out) *level_out = (int32_t)mx;
    return SCB_OK;
}

SCB_API scb_status scb_build_csr(const void* w, scb_dtype dt, const scb_shape* shape,
                                 int32_t unify, int64_t nnz_cap, void* values,
                                 int32_t* colidx, int32_t* rowptr) {
    Geom g;
    scb_status st = make_geom(shape, &g);
    if (st != SCB_OK) return st;
    int es = dtype_size(dt);
    if (!w || es == 0 || !rowptr) return fail(SCB_ERR_ARG, "bad arguments");
    if ((int64_t)g.c * g.hp * g.wp > 2147483647LL)
        return fail(SCB_ERR_SHAPE, "padded input volume exceeds 32-bit offset range");
    const int64_t vol = (int64_t)g.c * g.r * g.s;
    const int64_t rs = (int64_t)g.r * g.s;
    const int64_t plane = (int64_t)g.hp * g.wp;
    std::vector<int64_t> cnt(g.k);
    scb_channel_nnz(w, dt, g.k, vol, cnt.data());
    int64_t target = 0;
    for (int64_t v : cnt) target = std::max(target, v);
    const unsigned char* base = static_cast<const unsigned char*>(w);
    unsigned char* vout = static_cast<unsigned char*>(values);
    std::vector<int64_t> promoted;
    int64_t pos = 0;
    rowptr[0] = 0;
    for (int32_t ch = 0; ch < g.k; ++ch) {
        const unsigned char* row = base + (int64_t)ch * vol * es;
        if (unify && cnt[ch] < target) {
            if (!promote_zeros(row, es, vol, target - cnt[ch], promoted))
                return fail(SCB_ERR_SHAPE, "zero promotion failed");
        } else {
            promoted.clear();
        }
        // merge original nonzeros with the promoted zeros in index order
        size_t pi = 0;
        for (int64_t j = 0; j < vol; ++j) {
            bool take = !elem_is_zero(row + j * es, es);
            if (!take && pi < promoted.size() && promoted[pi] == j) { take = true; ++pi; }
            if (!take) continue;
            if (pos >= nnz_cap || !vout || !colidx) return fail(SCB_ERR_ARG, "nnz_cap too small");
            std::memcpy(vout + pos * es, row + j * es, es);
            int64_t c = j / rs, rem = j % rs;
            colidx[pos] = (int32_t)(c * plane + (rem / g.s) * g.wp + rem % g.s);
            ++pos;
        }
        rowptr[ch + 1] = (int32_t)pos;
    }
    return SCB_OK;
}

SCB_API scb_status scb_validate_csr(const scb_shape* shape, const int32_t* colidx,
                                    const int32_t* rowptr, int64_t nnz,
                                    int32_t unified, int32_t level) {
    Geom g;
    scb_status st = make_geom(shape, &g);
    if (st != SCB_OK) return st;
    if (!rowptr || (nnz > 0 && !colidx)) return fail(SCB_ERR_ARG, "NULL arrays");
    if (rowptr[0] != 0 || rowptr[g.k] != nnz)
        return fail(SCB_ERR_FORMAT, "rowptr must start at 0 and end at len(values)");
    for (int32_t ch = 0; ch < g.k; ++ch) {
        int32_t d = rowptr[ch + 1] - rowptr[ch];
        if (d < 0) return fail(SCB_ERR_FORMAT, "rowptr must be monotonically non-decreasing");
        if (unified && d != level) return fail(SCB_ERR_FORMAT, "unified kernel requires equal per-channel counts");
    }
    const int64_t plane = (int64_t)g.hp * g.wp;
    for (int64_t t = 0; t < nnz; ++t) {
        int64_t v = colidx[t];
        if (v < 0) return fail(SCB_ERR_FORMAT, "colidx entry outside the kernel volume");
        int64_t c = v / plane, rem = v % plane;
        if (c >= g.c || rem / g.wp >= g.r || rem % g.wp >= g.s)
            return fail(SCB_ERR_FORMAT, "colidx entry outside the kernel volume");
    }
    for (int32_t ch = 0; ch < g.k; ++ch)
        for (int32_t t = rowptr[ch] + 1; t < rowptr[ch + 1]; ++t)
            if (colidx[t] <= colidx[t - 1])
                return fail(SCB_ERR_FORMAT, "colidx not strictly increasing in channel " + std::to_string(ch));
    return SCB_OK;
}

SCB_API scb_status scb_decompress(const scb_shape* shape, scb_dtype dt, const void* values,
                                  const int32_t* colidx, const int32_t* rowptr,
                                  int64_t nnz, void* dense_out) {
    Geom g;
    scb_status st = make_geom(shape, &g);
    if (st != SCB_OK) return st;
    int es = dtype_size(dt);
    if (es == 0 || !dense_out || (nnz > 0 && (!values || !colidx)) || !rowptr)
        return fail(SCB_ERR_ARG, "bad arguments");
    const int64_t plane = (int64_t)g.hp * g.wp;
    const int64_t vol = (int64_t)g.c * g.r * g.s;
    std::memset(dense_out, 0, (size_t)(vol * g.k * es));
    const unsigned char* vin = static_cast<const unsigned char*>(values);
    unsigned char* d = static_cast<unsigned char*>(dense_out);
    for (int32_t ch = 0; ch < g.k; ++ch)
        for (int32_t t = rowptr[ch]; t < rowptr[ch + 1]; ++t) {
            int64_t c = colidx[t] / plane, rem = colidx[t] % plane;
            int64_t flat = (c * g.r + rem / g.wp) * g.s + rem % g.wp;
            std::memcpy(d + ((int64_t)ch * vol + flat) * es, vin + (int64_t)t * es, es);
        }
    return SCB_OK;
}

SCB_API const char* scb_last_error(void) { return g_last_error.c_str(); }

SCB_API const char* scb_version(void) { return "sparseconv_b200 0.1.0 (sm_100a)"; }

}  // extern "C"

extern "C" SCB_API scb_status scb_fnv1a64(const void* data, int64_t size, uint64_t* out) {
    if (!out || size < 0 || (size > 0 && !data)) return scb::fail(SCB_ERR_ARG, "fnv1a64: bad arguments");
    const unsigned char* p = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t i = 0; i < size; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
    *out = h;
    return SCB_OK;
}
