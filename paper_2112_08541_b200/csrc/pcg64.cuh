// PCG64 (numpy's PCG-XSL-RR 128/64, "setseq") replay on the device.
// Restated from numpy's published algorithm; oracle: oracle/pcg64.py.
#pragma once

#include <stdint.h>

namespace bgl {

struct U128 {
    uint64_t hi, lo;
};

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
    r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
    return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}

// s -> A*s + C
__host__ __device__ __forceinline__ U128 affine(U128 A, U128 C, U128 s) { return add128(mul128(A, s), C); }

// affine() with the 128-bit add as one add.cc/addc chain (no compare-and-
// select carry): the walk's per-draw step. In the walk loop it compiles to
// ~8 SASS instructions fewer than a 16-mad 32-bit-limb chain (whose ptxas
// expansion zeroes addends for every mad.hi) and ~2 fewer than affine().
__device__ __forceinline__ U128 affine_cc(U128 A, U128 C, U128 s) {
    const U128 p = mul128(A, s);
    uint32_t r0 = (uint32_t)p.lo, r1 = (uint32_t)(p.lo >> 32), r2 = (uint32_t)p.hi, r3 = (uint32_t)(p.hi >> 32);
    asm("add.cc.u32  %0, %0, %4;\n\t"
        "addc.cc.u32 %1, %1, %5;\n\t"
        "addc.cc.u32 %2, %2, %6;\n\t"
        "addc.u32    %3, %3, %7;"
        : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3)
        : "r"((uint32_t)C.lo), "r"((uint32_t)(C.lo >> 32)), "r"((uint32_t)C.hi), "r"((uint32_t)(C.hi >> 32)));
    return U128{((uint64_t)r3 << 32) | r2, ((uint64_t)r1 << 32) | r0};
}

// XSL-RR output of a (post-step) state.
__host__ __device__ __forceinline__ uint64_t xsl_rr(U128 s) {
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// xsl_rr with the 64-bit rotation as two 32-bit funnel shifts.
__device__ __forceinline__ uint64_t xsl_rr_fs(U128 s) {
    const uint32_t hh = (uint32_t)(s.hi >> 32);
    uint32_t xl = (uint32_t)s.lo ^ (uint32_t)s.hi, xh = (uint32_t)(s.lo >> 32) ^ hh;
    const uint32_t rot = hh >> 26;
    if (rot & 32u) {
        const uint32_t t = xl;
        xl = xh;
        xh = t;
    }
    const uint32_t lo = __funnelshift_r(xl, xh, rot), hi = __funnelshift_r(xh, xl, rot);
    return ((uint64_t)hi << 32) | lo;
}

// table layout: uint64 [kPcgTableRows][4]; row 0 = (state_hi, state_lo,
// inc_hi, inc_lo); row 1 + 15*i + (j-1) = (A_hi, A_lo, C_hi, C_lo) of the map
// advancing j * 16^i steps (i = 0..15, j = 1..15): a jump of delta steps is
// one affine map per nonzero hex digit of delta.
constexpr int kPcgTableRows = 1 + 16 * 15;

struct PcgTable {
    const uint64_t* t;
    __device__ __forceinline__ const uint64_t* row(int i, int j) const { return t + 4 * (1 + 15 * i + (j - 1)); }
    __device__ __forceinline__ U128 state() const { return U128{__ldg(t + 0), __ldg(t + 1)}; }
    // map advancing 2^k steps (k < 64)
    __device__ __forceinline__ U128 A(int k) const {
        const uint64_t* r = row(k >> 2, 1 << (k & 3));
        return U128{__ldg(r + 0), __ldg(r + 1)};
    }
    __device__ __forceinline__ U128 C(int k) const {
        const uint64_t* r = row(k >> 2, 1 << (k & 3));
        return U128{__ldg(r + 2), __ldg(r + 3)};
    }
    // State after `delta` steps from the stream start.
    __device__ __forceinline__ U128 at(uint64_t delta) const { return adv(state(), delta); }
    // s advanced by `delta` steps: one affine map per nonzero hex digit.
    __device__ __forceinline__ U128 adv(U128 s, uint64_t delta) const {
        while (delta) {
            const int i = (__ffsll((long long)delta) - 1) >> 2;
            const int j = (int)((delta >> (4 * i)) & 15u);
            const uint64_t* r = row(i, j);
            s = affine(U128{__ldg(r + 0), __ldg(r + 1)}, U128{__ldg(r + 2), __ldg(r + 3)}, s);
            delta &= ~(15ull << (4 * i));
        }
        return s;
    }
};

// 53-bit integer of draw number i (0-based): Generator.random() == m * 2^-53.
__device__ __forceinline__ uint64_t draw_of_state(U128 s) { return xsl_rr(s) >> 11; }

}  // namespace bgl
