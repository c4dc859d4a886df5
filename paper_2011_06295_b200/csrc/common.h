// Shared host/device helpers for the sparseconv_b200 library.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>

#include "sparseconv_b200.h"

namespace scb {

// Thread-local error message behind scb_last_error().
void set_error(const std::string& msg);
scb_status fail(scb_status code, const std::string& msg);

inline int dtype_size(scb_dtype dt) {
    switch (dt) {
        case SCB_F32: return 4;
        case SCB_F64: return 8;
        case SCB_F16: return 2;
    }
    return 0;
}

// IEEE zero test on a raw element (+0.0 and -0.0 are zero; NaN is not) --
// numpy count_nonzero / flatnonzero semantics used by csr.py:84,142.
inline bool elem_is_zero(const unsigned char* p, int esize) {
    if (esize == 2) { uint16_t v; std::memcpy(&v, p, 2); return (v & 0x7fffu) == 0; }
    if (esize == 4) { uint32_t v; std::memcpy(&v, p, 4); return (v & 0x7fffffffu) == 0; }
    uint64_t v; std::memcpy(&v, p, 8); return (v & 0x7fffffffffffffffull) == 0;
}

// ConvShape validation (shapes.py:35-51) + derived extents.
struct Geom {
    int n, c, h, w, k, r, s, stride, pad;
    int e, f, hp, wp;
};
scb_status make_geom(const scb_shape* sh, Geom* g);

}  // namespace scb
