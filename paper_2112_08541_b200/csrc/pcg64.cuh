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

// XSL-RR output of a (post-step) state.
__host__ __device__ __forceinline__ uint64_t xsl_rr(U128 s) {
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
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
    __device__ __forceinline__ U128 at(uint64_t delta) const {
        U128 s = state();
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
