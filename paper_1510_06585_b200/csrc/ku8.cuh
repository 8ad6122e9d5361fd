// ku8.cuh — the u8 chain's SWAR threshold primitives (segmentation /
// threshold / finalize), shared by the u8 chain kernels (chains.cu) and the
// bit-plane pack / unpack of the hysteresis (planes.cu).
#pragma once
#include "kcommon.cuh"

namespace mwk {
namespace {

// ------------------------------------------------------------ u8 chain (SWAR)
// Per-byte unsigned v >= c as bit 7 (c broadcast in every byte, 0 <= c <= 255).
__device__ __forceinline__ uint32_t ge_bytes(uint32_t x, uint32_t c7, bool c_hi) {
    // d bit7 = (x & 0x7f) >= (c & 0x7f); no inter-byte borrow since each byte of
    // (x | 0x80) - (c & 0x7f) is >= 1.
    uint32_t d = (x | 0x80808080u) - c7;
    return c_hi ? (x & d & 0x80808080u) : ((x | d) & 0x80808080u);
}
// threshold t in [0, 256]: mode 0 = every byte >= t (t <= 0), 1 = none (t >= 256),
// 2 = compare with t >= 128, 3 = compare with t < 128.
__device__ __forceinline__ uint32_t ge_t(uint32_t x, uint32_t c7, int mode) {
    return mode == 0 ? 0x80808080u : (mode == 1 ? 0u : ge_bytes(x, c7, mode == 2));
}
struct U8Const {
    uint32_t lo7[kMaxOps], hi7[kMaxOps];
    int32_t lo_mode[kMaxOps], hi_mode[kMaxOps];
};
__device__ __forceinline__ uint8_t apply_u8_byte(const U8Prog& p, uint8_t v) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT)
            v = v < p.lo[k] ? 0 : (v < p.hi[k] ? 128 : 255);
        else
            v = v == 128 ? 0 : v;
    }
    return v;
}

// Apply one SEGMENT op to N words with its threshold modes fixed at compile
// time (the per-op dispatch is hoisted out of the word loop).
template <int LM, int HM, int N>
__device__ __forceinline__ void seg_words(uint32_t* w, uint32_t lo7, uint32_t hi7) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const uint32_t x = w[i];
        const uint32_t flo = ge_t(x, lo7, LM), fhi = ge_t(x, hi7, HM);
        w[i] = flo | (fhi - (fhi >> 7));
    }
}
template <int N>
__device__ __forceinline__ void seg_dispatch(uint32_t* w, int lm, int hm, uint32_t lo7,
                                             uint32_t hi7) {
    switch (lm * 4 + hm) {
#define MW_SEG_CASE(A, B) \
    case A * 4 + B: seg_words<A, B, N>(w, lo7, hi7); break;
        MW_SEG_CASE(0, 0) MW_SEG_CASE(0, 1) MW_SEG_CASE(0, 2) MW_SEG_CASE(0, 3)
        MW_SEG_CASE(1, 1) MW_SEG_CASE(2, 1) MW_SEG_CASE(2, 2) MW_SEG_CASE(3, 1)
        MW_SEG_CASE(3, 2) MW_SEG_CASE(3, 3)
#undef MW_SEG_CASE
        default: break;   // unreachable for lo <= hi
    }
}

template <int N>
__device__ __forceinline__ void u8_apply_words(const U8Prog& p, const U8Const& c, uint32_t* w) {
    for (int k = 0; k < p.n; ++k) {
        if (p.kind[k] == U8_SEGMENT) {
            seg_dispatch<N>(w, c.lo_mode[k], c.hi_mode[k], c.lo7[k], c.hi7[k]);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                // R11 finalize: byte == 128 -> 0 (exact zero-byte test on x ^ 0x80)
                const uint32_t x = w[i];
                const uint32_t z = ~((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
                w[i] = x & ~((z >> 7) * 0xFFu);
            }
        }
    }
}


inline U8Const u8_consts(const U8Prog& p) {
    U8Const c;
    auto mode = [](int t) { return t <= 0 ? 0 : (t >= 256 ? 1 : (t >= 128 ? 2 : 3)); };
    for (int k = 0; k < p.n; ++k) {
        c.lo_mode[k] = mode(p.lo[k]);
        c.hi_mode[k] = mode(p.hi[k]);
        c.lo7[k] = (uint32_t)(p.lo[k] & 0x7F) * 0x01010101u;
        c.hi7[k] = (uint32_t)(p.hi[k] & 0x7F) * 0x01010101u;
    }
    return c;
}

// Batched device copies (halo rows between partitions on one device): one

}  // namespace
}  // namespace mwk
