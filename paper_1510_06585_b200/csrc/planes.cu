// planes.cu — the hysteresis Loop of Map (R11): the byte stencil and the bit-
// plane path (threshold fused into packing S / K planes, the whole while-loop
// in one cooperative kernel per rank — one or several partitions, across
// ranks through peer memory — per-pass kernels as the fallback, unpack fused
// with finalize).  The integer-ALU / shuffle-bound loop works on L2-resident
// planes; pack and unpack are HBM streams.
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
#include "kcommon.cuh"
#include "ku8.cuh"

namespace mwk {
namespace {

// ------------------------------------------------------------ hysteresis step
// R11: L'(p) = 255 if L(p) = 128 and an 8-neighbour inside the image is 255.
// Thread = 16-byte column segment x R rows; a warp covers 512 contiguous bytes
// of a row.  Rows slide through registers (prev/cur/next horizontal strong
// masks), so each input row is loaded once per strip (+2 halo rows / strip).
// Per-byte exact equality tests (SWAR): bit 7 of each byte.
__device__ __forceinline__ uint32_t is255(uint32_t x) {
    return ~((~x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
}
__device__ __forceinline__ uint32_t is128(uint32_t x) {
    return ~((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & x & 0x80808080u;
}

constexpr int kStencilRows = 32;
constexpr int kStencilThreads = 128;

struct Row4 {
    uint32_t w[4];
};

// strong mask of a row segment, OR-ed horizontally with its left/right bytes
__device__ __forceinline__ Row4 hmask(const uint4& v, uint32_t left_word, uint32_t right_word,
                                      int lane, bool lane_lo_edge, bool lane_hi_edge) {
    uint32_t s0 = is255(v.x), s1 = is255(v.y), s2 = is255(v.z), s3 = is255(v.w);
    // neighbouring words' strong masks across thread boundaries
    uint32_t up = __shfl_up_sync(0xffffffffu, s3, 1);     // lane-1's last word
    uint32_t dn = __shfl_down_sync(0xffffffffu, s0, 1);   // lane+1's first word
    if (lane == 0) up = is255(left_word);
    if (lane == 31) dn = is255(right_word);
    if (lane_lo_edge) up = 0;
    if (lane_hi_edge) dn = 0;
    Row4 h;
    h.w[0] = s0 | __funnelshift_l(up, s0, 8) | __funnelshift_r(s0, s1, 8);
    h.w[1] = s1 | __funnelshift_l(s0, s1, 8) | __funnelshift_r(s1, s2, 8);
    h.w[2] = s2 | __funnelshift_l(s1, s2, 8) | __funnelshift_r(s2, s3, 8);
    h.w[3] = s3 | __funnelshift_l(s2, s3, 8) | __funnelshift_r(s3, dn, 8);
    return h;
}

// Active-tile Jacobi: a tile whose 3x3 tile neighbourhood changed nothing
// in the previous execution is already at the next state in the output
// buffer (state_{k-1} == state_k == state_{k+1} there), so it is skipped —
// the iterates, the fixed point and E are exactly those of dense Jacobi.
// prev_flags == nullptr: every tile is active (first execution).
__global__ void __launch_bounds__(kStencilThreads) k_hyst_step(
    const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t rows, int64_t pitch,
    int iter, int* last_changed, int64_t n_strips, int64_t n_colblk,
    const uint8_t* __restrict__ prev_flags, uint8_t* __restrict__ cur_flags, int top_nbr,
    int bot_nbr) {
    const int lane = threadIdx.x & 31;
    const int64_t segs = pitch >> 4;  // 16-byte segments per row
    const int64_t n_tiles = n_strips * n_colblk;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t strip = t / n_colblk, cb = t - strip * n_colblk;
        bool active = prev_flags == nullptr || (top_nbr && strip == 0) ||
                      (bot_nbr && strip == n_strips - 1);
        if (!active) {
            for (int64_t ds = -1; ds <= 1 && !active; ++ds)
                for (int64_t dc = -1; dc <= 1; ++dc) {
                    const int64_t s2 = strip + ds, c2 = cb + dc;
                    if (s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_colblk &&
                        prev_flags[s2 * n_colblk + c2]) {
                        active = true;
                        break;
                    }
                }
        }
        if (!active) {   // uniform over the CTA
            if (threadIdx.x == 0) cur_flags[t] = 0;
            continue;
        }
        uint32_t changed = 0;
        const int64_t seg = cb * kStencilThreads + threadIdx.x;
        const bool valid = seg < segs;
        const int64_t y0 = strip * kStencilRows;                 // first interior row
        const int64_t y1 = min(rows, y0 + (int64_t)kStencilRows);
        const bool lo_edge = seg == 0, hi_edge = seg == segs - 1;
        // row pointer for interior row y (halo rows are y = -1 and y = rows)
        auto rowp = [&](int64_t y) { return in + (y + 1) * pitch; };
        auto load = [&](int64_t y, uint32_t& lw, uint32_t& rw) {
            const uint8_t* r = rowp(y);
            uint4 v = valid ? *reinterpret_cast<const uint4*>(r + seg * 16) : make_uint4(0, 0, 0, 0);
            lw = (lane == 0 && valid && !lo_edge) ? *reinterpret_cast<const uint32_t*>(r + seg * 16 - 4) : 0u;
            rw = (lane == 31 && valid && !hi_edge) ? *reinterpret_cast<const uint32_t*>(r + seg * 16 + 16) : 0u;
            return v;
        };
        uint32_t lw, rw;
        uint4 vprev = load(y0 - 1, lw, rw);
        Row4 hprev = hmask(vprev, lw, rw, lane, lo_edge, hi_edge);
        uint4 vcur = load(y0, lw, rw);
        Row4 hcur = hmask(vcur, lw, rw, lane, lo_edge, hi_edge);
        for (int64_t y = y0; y < y1; ++y) {
            uint4 vnext = load(y + 1, lw, rw);
            Row4 hnext = hmask(vnext, lw, rw, lane, lo_edge, hi_edge);
            uint32_t c[4] = {vcur.x, vcur.y, vcur.z, vcur.w};
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t prom = is128(c[k]) & (hprev.w[k] | hcur.w[k] | hnext.w[k]);
                changed |= prom;
                o[k] = c[k] + (prom >> 7) * 0x7Fu;   // 0x80 -> 0xFF where promoted
            }
            if (valid)
                *reinterpret_cast<uint4*>(out + (y + 1) * pitch + seg * 16) =
                    make_uint4(o[0], o[1], o[2], o[3]);
            vcur = vnext;
            hprev = hcur;
            hcur = hnext;
        }
        const int tile_changed = __syncthreads_or(changed != 0);
        if (threadIdx.x == 0) {
            cur_flags[t] = (uint8_t)tile_changed;
            if (tile_changed) atomicMax(last_changed, iter);
        }
    }
}

// ------------------------------------------------------------ hysteresis on bit planes
// When the labels entering the loop are known to be 3-valued (the stage
// before the loop ends with the threshold), the loop state is held as two
// bit planes: S (== 255) and K (== 128, constant).  One Jacobi execution is
//     S' = S | (K & dilate8(S))
// on 32 pixels per 32-bit word — the same iterates as the byte stencil, at
// 1/16 of the bytes (the 16384^2 planes are 32 MiB each and stay in L2).
// The whole while-loop runs in ONE cooperative kernel: the loop condition is
// evaluated on the device after a grid-wide barrier every execution (exact,
// no extra executions, no host round trip).  Plane layout: (rows + 2) x wp
// words, rows 0 and rows+1 zero halos; bit b of word w is pixel x = 32w + b.

__device__ __forceinline__ uint32_t nib_of(uint32_t flags80) {   // bits 7,15,23,31 -> 4 bits
    return ((flags80 >> 7) * 0x10204080u) >> 28;
}
__device__ __forceinline__ uint32_t expand_nib(uint32_t n) {      // 4 bits -> 0x00/0xFF bytes
    return ((n * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// SEG >= 0: the chain is exactly one threshold with compile-time compare modes
// (lo mode = SEG / 4, hi mode = SEG % 4); SEG < 0: any chain ending with it.
// blockIdx.y = partition (PlaneIO table: several partitions in one launch)
template <int SEG>
__global__ void __launch_bounds__(256) k_planes_pack(const __grid_constant__ U8Prog p,
                                                     const __grid_constant__ U8Const c,
                                                     const __grid_constant__ PlaneIO io, int64_t W,
                                                     int64_t wp, FastDiv WP, int hd) {
    const int q = blockIdx.y;
    const uint8_t* __restrict__ src = io.src[q];
    const int64_t sp = io.sp;
    uint32_t* __restrict__ S = io.S0[q];
    uint32_t* __restrict__ K = io.K[q];
    const uint32_t total = (uint32_t)(io.rows[q] * wp);
    uint32_t one;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(one));
    one = one > 0u ? 1u : 0u;
    for (uint32_t n = blockIdx.x * 256u + threadIdx.x; n < total; n += gridDim.x * 256u) {
        const uint32_t y = fdiv(n, WP), w = n - y * WP.d;
        const int64_t x0 = 32ll * w;
        const uint8_t* r = src + y * sp + x0;
        uint32_t v[8];
        if (x0 + 32 <= W && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
            const uint4 a = ld_stream(reinterpret_cast<const uint4*>(r));
            const uint4 b = ld_stream(reinterpret_cast<const uint4*>(r) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t x = 0;
                for (int e = 0; e < 4; ++e) {
                    const int64_t xx = x0 + 4 * i + e;
                    if (xx < W) x |= (uint32_t)r[4 * i + e] << (8 * e);
                }
                v[i] = x;
            }
        }
        uint32_t sb = 0, kb = 0;
        if constexpr (SEG >= 0) {
            // the chain is exactly the threshold: strong = v >= hi, weak = lo <= v < hi.
            // The byte msbs 7,15,23,31 land on product bits 28..31 of f * 0x00204081
            // (partial products at distinct bits: no carries), then move to 4i.
            // The nibble lands at bit 4i through a multiply-add by 2^(4i) (FMA
            // pipe; the nibbles are disjoint) — `one` is opaque to ptxas
            // (%nsmid >= 1) so it stays an IMAD instead of a shift + OR.
            // lo <= hi, so the strong flags are a subset of the v >= lo flags:
            // weak = (v >= lo) - strong, bitwise and as whole planes.
            const uint32_t l7 = c.lo7[0], h7 = c.hi7[0];
            uint32_t lb = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t fhi = ge_t(v[i], h7, SEG % 4), flo = ge_t(v[i], l7, SEG / 4);
                const uint32_t pw = one << (4 * i);
                sb = ((fhi * 0x00204081u) >> 28) * pw + sb;
                lb = ((flo * 0x00204081u) >> 28) * pw + lb;
            }
            kb = lb - sb;
        } else {
            u8_apply_words<8>(p, c, v);   // the chain before the loop (ends with the threshold)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                sb |= nib_of(is255(v[i])) << (4 * i);
                kb |= nib_of(is128(v[i])) << (4 * i);
            }
        }
        const int64_t rem = W - x0;   // bits beyond the image width stay 0
        if (rem < 32) {   // (pad words past the image: rem <= 0)
            const uint32_t keep = rem <= 0 ? 0u : (1u << rem) - 1u;
            sb &= keep;
            kb &= keep;
        }
        S[(y + hd) * wp + w] = sb;
        K[(y + hd) * wp + w] = kb;
    }
}

// Unpack when the chain after the loop is exactly finalize and a row has a
// multiple of 4096 pixels: a warp owns 4 KiB of output (128 plane words);
// lane l writes 16-byte chunk l of every 512 B, so each STG.128 of the warp
// covers 512 contiguous bytes, and the 8 plane-word loads per lane (2 lanes
// share a word) are issued before any store.  (The per-word variant below
// left every thread with one dependent L2 load per 32 bytes of output.)
__global__ void __launch_bounds__(256) k_planes_unpack_fin_w(const __grid_constant__ PlaneIO io,
                                                             const int* __restrict__ state,
                                                             int64_t dp, int64_t wp, FastDiv UPR,
                                                             int hd) {
    const int q = blockIdx.y;
    const uint32_t* S = state[2] ? io.S1[q] : io.S0[q];
    uint8_t* __restrict__ dst = io.dst[q];
    const int lane = threadIdx.x & 31;
    const uint32_t total = (uint32_t)(io.rows[q] * (wp / 128));
    for (uint32_t u = blockIdx.x * 8u + (threadIdx.x >> 5); u < total; u += gridDim.x * 8u) {
        const uint32_t y = fdiv(u, UPR), q = u - y * UPR.d;
        const uint32_t* srow = S + ((int64_t)y + hd) * wp + 128ll * q;
        uint8_t* drow = dst + (int64_t)y * dp + 4096ll * q + 16 * lane;
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = srow[(lane >> 1) + 16 * k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t h = w[k] >> (16 * (lane & 1));   // this lane's 16 pixels
            uint32_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t m = ((h >> (4 * i)) & 15u) * 0x10204080u;
                asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(v[i]) : "r"(m));
            }
            st_stream(reinterpret_cast<uint4*>(drow + 512 * k), make_uint4(v[0], v[1], v[2], v[3]));
        }
    }
}

template <bool FIN_ONLY>
__global__ void __launch_bounds__(256) k_planes_unpack(const __grid_constant__ U8Prog p,
                                                       const __grid_constant__ U8Const c,
                                                       const __grid_constant__ PlaneIO io,
                                                       const int* __restrict__ state, int64_t dp,
                                                       int64_t W, int64_t wp, FastDiv WP, int hd) {
    const int q = blockIdx.y;
    const uint32_t* S = state[2] ? io.S1[q] : io.S0[q];
    const uint32_t* __restrict__ K = io.K[q];
    uint8_t* __restrict__ dst = io.dst[q];
    const uint32_t total = (uint32_t)(io.rows[q] * wp);
    for (uint32_t n = blockIdx.x * 256u + threadIdx.x; n < total; n += gridDim.x * 256u) {
        const uint32_t y = fdiv(n, WP), w = n - y * WP.d;
        const uint32_t sb = S[(y + hd) * wp + w];
        uint32_t v[8];
        if (FIN_ONLY) {
            // the chain is exactly finalize (128 -> 0): strong pixels 255, all else 0;
            // nibble bits to byte msbs with one IMAD, then a sign-replicating PRMT
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t m = ((sb >> (4 * i)) & 15u) * 0x10204080u;
                asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(v[i]) : "r"(m));
            }
        } else {
            const uint32_t kb = K[(y + hd) * wp + w];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t bs = expand_nib((sb >> (4 * i)) & 15u);
                const uint32_t bk = expand_nib((kb >> (4 * i)) & 15u);
                v[i] = bs | (bk & 0x80808080u);   // 255 / 128 / 0 labels
            }
            u8_apply_words<8>(p, c, v);           // the chain after the loop
        }
        const int64_t x0 = 32ll * w;
        uint8_t* r = dst + y * dp + x0;
        if (x0 + 32 <= W && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
            st_stream(reinterpret_cast<uint4*>(r), make_uint4(v[0], v[1], v[2], v[3]));
            st_stream(reinterpret_cast<uint4*>(r) + 1, make_uint4(v[4], v[5], v[6], v[7]));
        } else {
            for (int e = 0; e < 32 && x0 + e < W; ++e) r[e] = (uint8_t)(v[e >> 2] >> (8 * (e & 3)));
        }
    }
}

// Temporal blocking: one pass advances the state by T Jacobi executions.  A
// warp tile holds kTbRows rows x 32 words in registers: lanes 1..30 and rows
// T..kTbRows-T-1 are owned (written back), lanes 0/31 and T rows above and
// below are halo recomputed from the neighbours (validity shrinks by one
// pixel per execution, so T <= 31 bits / T <= kTbRows/2 rows stay exact).
// Every execution inside a pass is one global Jacobi step; the device keeps
// the last execution index that changed an owned pixel, so E is exact and a
// pass that ends without change has reached the fixed point (extra in-pass
// executions past it are no-ops).  Tiles are skipped when provably unchanged
// (no live front in their 3x3 tile neighbourhood and no change of their own in
// the previous pass; DESIGN R35), and a tile stops its pass early once an
// execution changes nothing on its exact positions (R34).  One cooperative
// kernel runs all passes; flags[pass % 3] = last changed execution of the
// pass (-1: none).

// One warp tile: T Jacobi executions (steps <= T) on register rows
// [strip*R - T, strip*R + R + T) x lanes, owned rows/lanes written to `out`.
// Buffers hold rows [-hd, rows + hd) at buffer row y + hd (halo rows: zero at
// the image boundary, the neighbour partition's rows otherwise); rows outside
// are zero.  Returns the last execution (0-based) that changed an owned bit.
// (Measured on B200: keeping the weak plane in registers with 256-thread CTAs
// and a rolled execution loop beats smem-resident K and a fully unrolled
// shrinking-window loop, whose code no longer fits the instruction cache.)

// One execution on register rows [LO, HI] (rows outside keep their values
// and only serve as neighbours).  Returns bit 0: an owned row [T, ROWS - T)
// of an owned lane changed; bit 1: a bit of the window inside `vm` changed.
// vm masks off the bits of lanes 0/31 whose value is no longer exact (their
// missing outer neighbour: one bit per execution from the far end).
template <int T, int ROWS, int LO, int HI>
__device__ __forceinline__ int plane_exec(uint32_t (&sv)[ROWS], const uint32_t (&kv)[ROWS],
                                          bool own_lane, uint32_t vm) {
    auto hrow = [&](uint32_t sx) {
        // lanes 0/31 take their own word as the outer neighbour: the error
        // enters at their far bits and moves one bit per execution, never
        // reaching the owned lanes (T <= 16)
        const uint32_t l = __shfl_up_sync(0xffffffffu, sx, 1);
        const uint32_t r = __shfl_down_sync(0xffffffffu, sx, 1);
        return sx | __funnelshift_l(l, sx, 1) | __funnelshift_r(sx, r, 1);
    };
    uint32_t hp = hrow(sv[LO - 1]), hc = hrow(sv[LO]);
    uint32_t ch = 0, ca = 0;
#pragma unroll
    for (int i = LO; i <= HI; ++i) {
        const uint32_t hn = hrow(sv[i + 1]);     // old row i+1 (not yet updated)
        const uint32_t s2 = sv[i] | (kv[i] & (hp | hc | hn));
        if (i >= T && i < ROWS - T) ch |= s2 ^ sv[i];
        else ca |= s2 ^ sv[i];
        sv[i] = s2;
        hp = hc;
        hc = hn;
    }
    const bool any = ((ch | ca) & vm) != 0;
    return (__any_sync(0xffffffffu, own_lane && ch != 0) ? 1 : 0) | (__any_sync(0xffffffffu, any) ? 2 : 0);
}

// T executions on a register tile (rows [ybase, ybase + ROWS) x lanes).
// Row r is exact after execution st when st < r < ROWS - 1 - st (validity
// shrinks by a row per execution at each end), so a full pass computes rows
// [1, ROWS-2] in its first T/2 executions and only [T/2 + 1, ROWS - 2 - T/2]
// in the rest (a superset of what each later execution needs); executions
// run in pairs so the updated rows alternate between two register sets
// instead of being moved back every execution.
// Early stop: the positions still exact after execution j+1 shrink by the
// stencil radius per execution (V_{j+1} within V_j), and their values depend
// only on V_j.  When execution j+1 changes nothing on (a superset of) V_{j+1},
// the true iterates j and j+1 agree there, hence by induction every later
// iterate agrees with iterate j on the smaller V_m, which contains the owned
// region: the remaining executions of the pass cannot change an owned bit,
// and the registers already hold the pass's result there.
// Returns the last execution (0-based) that changed an owned bit.
template <int T, int ROWS>
__device__ __forceinline__ int plane_steps(uint32_t (&sv)[ROWS], const uint32_t (&kv)[ROWS],
                                           int steps, bool own_lane, int lane, int* nexec = nullptr) {
    int tile_last = -1;
    int ne = 0;
    struct Cnt {   // executions run (diagnostics: MW_HYST_PROF)
        int* p; int& n;
        __device__ ~Cnt() { if (p) *p = n; }
    } cnt{nexec, ne};
    // exact bits of this lane after the next execution (lanes 0/31 lose one
    // bit per execution at their far end)
    const int shl = lane == 0, shr = lane == 31;
    uint32_t vm = ~0u;
    if (T % 4 == 0 && steps == T) {
        constexpr int H = T / 2;
#pragma unroll 1
        for (int st = 0; st < H; st += 2) {
            vm = (vm << shl) >> shr;
            ++ne;
            int r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st;
            if (!(r & 2)) return tile_last;
            vm = (vm << shl) >> shr;
            ++ne;
            r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st + 1;
            if (!(r & 2)) return tile_last;
        }
#pragma unroll 1
        for (int st = H; st < T; st += 2) {
            vm = (vm << shl) >> shr;
            ++ne;
            int r = plane_exec<T, ROWS, H + 1, ROWS - 2 - H>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st;
            if (!(r & 2)) return tile_last;
            vm = (vm << shl) >> shr;
            ++ne;
            r = plane_exec<T, ROWS, H + 1, ROWS - 2 - H>(sv, kv, own_lane, vm);
            if (r & 1) tile_last = st + 1;
            if (!(r & 2)) return tile_last;
        }
        return tile_last;
    }
#pragma unroll 1
    for (int st = 0; st < steps; ++st) {
        vm = (vm << shl) >> shr;
        ++ne;
        const int r = plane_exec<T, ROWS, 1, ROWS - 2>(sv, kv, own_lane, vm);
        if (r & 1) tile_last = st;
        if (!(r & 2)) break;
    }
    return tile_last;
}

template <int T, int ROWS>
__device__ __forceinline__ void plane_store(const uint32_t (&sv)[ROWS], uint32_t* __restrict__ out,
                                            int64_t rows, int64_t wp, int hd, int64_t ybase,
                                            int64_t w, bool own_lane, bool wv) {
    constexpr int R = ROWS - 2 * T;
    if (!own_lane || !wv) return;
    uint32_t* o = out + (ybase + T + hd) * wp + w;    // owned row 0
    const uint32_t pw = (uint32_t)wp;
    if (ybase + T + R <= rows) {                       // every owned row inside the image
#pragma unroll
        for (int i = 0; i < R; ++i) o[i * pw] = sv[T + i];
    } else {
        const int n = (int)(rows - (ybase + T));
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (i < n) o[i * pw] = sv[T + i];
    }
}

// is tile t active: some tile of its 3x3 neighbourhood changed in the last
// execution of the previous pass (flag bit 0), the tile itself changed at any
// execution of it (bit 1: its newest state must reach this pass's output
// buffer), or it touches a partition boundary whose halo may have changed.
// A front that stopped before the last execution of a pass changes nothing
// later, and one alive at it moves at most T pixels in the next pass, which
// stays inside the 3x3 tile neighbourhood (T <= R rows, T <= 30 words).
__device__ __forceinline__ bool plane_tile_active(const uint8_t* fprev, int64_t strip, int64_t cb,
                                                  int64_t n_strips, int64_t n_cb, bool first,
                                                  int top_nbr, int bot_nbr, int lane) {
    bool act = first || (top_nbr && strip == 0) || (bot_nbr && strip == n_strips - 1);
    if (!act) {
        bool a = false;
        if (lane < 9) {
            const int64_t s2 = strip + lane / 3 - 1, c2 = cb + lane % 3 - 1;
            a = s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_cb &&
                (fprev[s2 * n_cb + c2] & (lane == 4 ? 3 : 1));
        }
        act = __any_sync(0xffffffffu, a);
    }
    return act;
}

// Whole loop, one partition per device: one cooperative kernel, all passes.
// Every warp prefetches its next active tile (S and K boxes of ROWS x 36
// words from the 16-byte-aligned column at or left of the tile's first word
// — TMA box origins are 16-byte aligned; lane l reads word o + l of a box
// row — 2-D TMA with out-of-bounds zero fill = the image-boundary rule)
// into one of its two shared-memory slots while it computes the current one;
// the L2 latency of the tile load (~2.4 us per tile measured with plain
// loads, 28 % of the loop in round 1) is hidden behind the executions.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// One pass of a warp over its tiles (t = gw, gw + nwarps, ...): prefetch the
// next active tile into the warp's slot (sb: S box, kb: K box, bar, phase)
// while the current one runs its executions; returns the last execution
// (0-based) in which one of the warp's tiles changed an owned bit.  Buffers
// hold rows [-hd, rows + hd) at buffer row y + hd; tensor maps cover them.
template <int T, int ROWS>
__device__ __forceinline__ int plane_pass_warp(const CUtensorMap* tin, const CUtensorMap* tk,
                                               uint32_t* __restrict__ out, int64_t rows,
                                               int64_t wp, int hd, int steps,
                                               const uint8_t* __restrict__ fprev,
                                               uint8_t* __restrict__ fcur, bool all_active,
                                               int top_nbr, int bot_nbr, int64_t gw,
                                               int64_t nwarps, int lane, uint32_t* sb,
                                               uint32_t* kb, uint64_t* bar, uint32_t& phase,
                                               bool last_bit = false,
                                               unsigned long long* pstat = nullptr) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;                          // box width (words)
    constexpr uint32_t kBox = ROWS * BW * 4;        // bytes per plane box
    const int64_t n_strips = (rows + R - 1) / R;
    const int64_t n_cb = (wp + OW - 1) / OW;
    const int64_t n_tiles = n_strips * n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    // the next active tile of this warp at or after t (inactive ones are
    // marked unchanged on the way)
    auto next_active = [&](int64_t t) {
        for (; t < n_tiles; t += nwarps) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            if (plane_tile_active(fprev, strip, cb, n_strips, n_cb, all_active, top_nbr, bot_nbr, lane))
                break;
            if (lane == 0) fcur[t] = 0;
        }
        return t;
    };
    auto issue = [&](int64_t t) {
        if (lane == 0) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R - T + hd);
            mbar_expect_tx(bar, 2 * kBox);
            tma_load_2d(sb, tin, x, y, bar);
            tma_load_2d(kb, tk, x, y, bar);
        }
    };
    int my_last = -1;
    int64_t t = next_active(gw);
    if (t < n_tiles) issue(t);
    while (t < n_tiles) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        const int o = (int)((t % n_cb) * OW - 1) & 3;   // tile's first word in the box
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                               // slot free: prefetch the next tile
        const int64_t tn = next_active(t + nwarps);
        if (tn < n_tiles) issue(tn);
        const int64_t strip = t / n_cb, cb = t - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        int ne = 0;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane, pstat ? &ne : nullptr);
        if (pstat && lane == 0) {
            atomicAdd(pstat, (unsigned long long)ne);
            atomicAdd(pstat + 32, 1ull);
        }
        // bit 0: changed in the last execution of the pass (fronts still alive);
        // bit 1: changed at all.  last_bit = false: bit 0 = bit 1 (the looser
        // any-change rule; both kernels use the tight one — boundary strips of
        // a partition with a neighbour are active every pass regardless).
        const uint8_t fl = tl < 0 ? 0 : (tl == steps - 1 || !last_bit ? 3 : 2);
        my_last = max(my_last, tl);
        plane_store<T, ROWS>(sv, out, rows, wp, hd, strip * R - T, w, own_lane, w >= 0 && w < wp);
        if (lane == 0) fcur[t] = fl;
        t = tn;
    }
    return my_last;
}

// The per-warp slots of shared memory: [8][2][ROWS][36] words, then 8 mbarriers.
template <int ROWS>
constexpr size_t plane_smem_bytes() { return 8 * 2 * ROWS * 36 * 4 + 8 * 8; }
// The one-partition loop keeps TWO slots per warp: [8][2 slots][2][ROWS][36]
// words, then 16 mbarriers (221 KiB at ROWS = 48).
template <int ROWS>
constexpr size_t plane_loop_smem_bytes() { return 8 * 2 * 2 * ROWS * 36 * 4 + 16 * 8; }

// One pass of the one-partition loop for one warp.  Activity is PUSHED: a
// tile that changed an owned bit stamps itself for the next pass (its newest
// state must reach the other buffer), and one still changing in the last
// execution (a live front, which moves at most T <= R rows / 30 words in the
// next pass) stamps its 3x3 tile neighbourhood.  act[t] == stamp: t is
// active in this pass (stamps are unique per pass and run, so nothing is ever
// cleared; a stale equal value could only add work, never change a result:
// a processed tile computes the same iterates from the buffer).  The warp
// reads the stamps of its tiles (gw + i nwarps) 32 at a time, so the active
// list is known up front (no per-tile flag scan on the critical path), and
// keeps two tiles in flight in its two slots — in the sparse late passes a
// tile runs 1-2 executions, too few to hide a tile load behind.  (Measured:
// a global queue of the pass's active tiles claimed with atomics — dynamic
// balance — made every pass ~2x slower: one hot counter for ~10^4 claims.)
template <int T, int ROWS>
__device__ __forceinline__ int plane_loop_pass_warp(const CUtensorMap* tin, const CUtensorMap* tk,
                                                    uint32_t* __restrict__ out, int64_t rows,
                                                    int64_t wp, int steps, uint32_t* __restrict__ act,
                                                    uint32_t stamp, bool all_active, int64_t gw,
                                                    int64_t nwarps, int lane, uint32_t* slots,
                                                    uint64_t* bars, uint32_t& phases,
                                                    unsigned long long* pstat) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;
    constexpr uint32_t kBox = ROWS * BW * 4;
    const int64_t n_strips = (rows + R - 1) / R;
    const int64_t n_cb = (wp + OW - 1) / OW;
    const int64_t n_tiles = n_strips * n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    const int64_t n_my = gw < n_tiles ? (n_tiles - gw + nwarps - 1) / nwarps : 0;
    // active-tile generator over the warp's tiles, 32 stamps per load
    int64_t chunk = -1;
    uint32_t mask = 0;
    auto next_tile = [&]() -> int64_t {
        while (mask == 0) {
            ++chunk;
            if (chunk * 32 >= n_my) return -1;
            const int64_t i = chunk * 32 + lane;
            bool a = false;
            if (i < n_my) a = all_active || __ldcg(act + gw + i * nwarps) == stamp;
            mask = __ballot_sync(0xffffffffu, a);
        }
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        return gw + (chunk * 32 + b) * nwarps;
    };
    auto issue = [&](int64_t t, int s) {
        if (lane == 0) {
            const int64_t strip = t / n_cb, cb = t - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R - T + 1);   // hd = 1
            uint32_t* sb = slots + s * (2 * ROWS * BW);
            mbar_expect_tx(&bars[s], 2 * kBox);
            tma_load_2d(sb, tin, x, y, &bars[s]);
            tma_load_2d(sb + ROWS * BW, tk, x, y, &bars[s]);
        }
    };
    int my_last = -1;
    int64_t cur = next_tile();
    if (cur >= 0) issue(cur, 0);
    int64_t nxt = cur >= 0 ? next_tile() : -1;
    if (nxt >= 0) issue(nxt, 1);
    int s = 0;
    while (cur >= 0) {
        mbar_wait(&bars[s], (phases >> s) & 1u);
        phases ^= 1u << s;
        const uint32_t* sb = slots + s * (2 * ROWS * BW);
        const uint32_t* kb = sb + ROWS * BW;
        const int o = (int)((cur % n_cb) * OW - 1) & 3;
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                                  // slot s free: refill it
        const int64_t n2 = nxt >= 0 ? next_tile() : -1;
        if (n2 >= 0) issue(n2, s);
        const int64_t strip = cur / n_cb, cb = cur - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        int ne = 0;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane, pstat ? &ne : nullptr);
        if (pstat && lane == 0) {
            atomicAdd(pstat, (unsigned long long)ne);
            atomicAdd(pstat + 32, 1ull);
        }
        my_last = max(my_last, tl);
        plane_store<T, ROWS>(sv, out, rows, wp, 1, strip * R - T, w, own_lane, w >= 0 && w < wp);
        if (tl >= 0) {
            const int64_t s2 = strip + lane / 3 - 1, c2 = cb + lane % 3 - 1;
            const bool nb = tl == steps - 1 ? lane < 9 : lane == 4;
            if (nb && s2 >= 0 && s2 < n_strips && c2 >= 0 && c2 < n_cb) act[s2 * n_cb + c2] = stamp + 1;
        }
        cur = nxt;
        nxt = n2;
        s ^= 1;
    }
    return my_last;
}

template <int T, int ROWS>
__global__ void __launch_bounds__(256) k_planes_loop(const __grid_constant__ CUtensorMap tm_s0,
                                                     const __grid_constant__ CUtensorMap tm_s1,
                                                     const __grid_constant__ CUtensorMap tm_k,
                                                     uint32_t* __restrict__ S0,
                                                     uint32_t* __restrict__ S1, int64_t rows,
                                                     int64_t wp, int64_t max_iters,
                                                     int* __restrict__ flags,
                                                     int* __restrict__ state,
                                                     uint32_t* __restrict__ act,
                                                     unsigned long long* __restrict__ prof) {
    constexpr int R = ROWS - 2 * T;
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];   // 8 x 2 warp slots, then 16 mbarriers
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * 2 * ROWS * BW);
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* slots = psm + wid * (2 * 2 * ROWS * BW);
    uint64_t* bar = &bars[2 * wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const int64_t n_tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    // act[n_tiles] = this run's stamp base (pass p is active at base + p);
    // the leader advances it past the run's stamps after the last barrier
    const uint32_t base = *((volatile uint32_t*)&act[n_tiles]);
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    if (prof && leader) prof[0] = gtime();
    uint32_t phases = 0;
    int64_t k0 = 0;
    int pass = 0;
    while (k0 < max_iters) {
        const int steps = (int)min((int64_t)T, max_iters - k0);
        if (leader) flags[(pass + 1) % 3] = -1;   // last read two barriers ago
        const int my_last = plane_loop_pass_warp<T, ROWS>(
            (pass & 1) ? &tm_s1 : &tm_s0, &tm_k, (pass & 1) ? S0 : S1, rows, wp, steps, act,
            base + (uint32_t)pass, pass == 0, gw, nwarps, lane, slots, bar, phases,
            prof && pass < 30 ? prof + 32 + pass : nullptr);
        if (lane == 0 && my_last >= 0) atomicMax(&flags[pass % 3], (int)(k0 + my_last));
        // the next pass reads `out` through the async (TMA) proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        grid.sync();
        if (prof && leader) prof[1 + pass] = gtime();
        const int last = *((volatile int*)&flags[pass % 3]);
        if (last < k0 + steps - 1) {   // the pass ended with an execution that changed nothing
            if (leader) {
                const int64_t last_global = last >= 0 ? last : k0 - 1;
                state[0] = (int)(last_global + 2);
                state[1] = 1;
                state[2] = (pass & 1) ? 0 : 1;
                act[n_tiles] = base + (uint32_t)pass + 2;
                // ready for the next run (every thread has read the flags
                // and decided to leave: -1 only confirms that decision)
                flags[0] = -1;
            }
            return;
        }
        k0 += steps;
        ++pass;
    }
    if (leader) {
        state[0] = (int)max_iters;
        state[1] = 0;
        state[2] = pass == 0 ? 0 : (((pass - 1) & 1) ? 0 : 1);
        act[n_tiles] = base + (uint32_t)pass + 2;
        flags[0] = -1;
    }
}

// One pass over one partition of several (halo depth T, host loop between
// passes exchanges T plane rows with the neighbours and reduces `last`);
// the same TMA-prefetched warp tiles as the one-partition loop.
template <int T, int ROWS>
__global__ void __launch_bounds__(256) k_planes_pass(const __grid_constant__ CUtensorMap tm_in,
                                                     const __grid_constant__ CUtensorMap tm_k,
                                                     uint32_t* __restrict__ out, int64_t rows,
                                                     int64_t wp, int steps, int64_t k0,
                                                     const uint8_t* __restrict__ fprev,
                                                     uint8_t* __restrict__ fcur, int first,
                                                     int top_nbr, int bot_nbr,
                                                     int* __restrict__ last) {
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * ROWS * BW);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* sb = psm + wid * (2 * ROWS * BW);
    uint32_t* kb = sb + ROWS * BW;
    uint64_t* bar = &bars[wid];
    if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;
    const int my_last = plane_pass_warp<T, ROWS>(
        &tm_in, &tm_k, out, rows, wp, T, steps, fprev, fcur, first != 0, top_nbr, bot_nbr,
        (int64_t)blockIdx.x * 8 + wid, (int64_t)gridDim.x * 8, lane, sb, kb, bar, phase, true);
    if (lane == 0 && my_last >= 0) atomicMax(last, (int)(k0 + my_last));
}

// Whole loop over SEVERAL partitions of one rank in one cooperative kernel.
// The partitions keep their own plane buffers with T halo rows (the layout
// of the per-pass protocol); the global tile list is the concatenation of the
// partitions' tiles.  The halo exchange between neighbouring partitions is
// folded into the store: a tile writing owned rows y < T (y >= rows - T) of
// partition q also writes them into the bottom (top) halo rows of the previous
// (next) active partition's output buffer — a pointer table, no extra pass
// and no extra barrier; the next pass reads them through TMA after the grid
// barrier.  Loop condition and exact E as in k_planes_loop.
template <int T, int ROWS>
__device__ __forceinline__ void plane_store_fwd(const uint32_t (&sv)[ROWS], const PlaneMultiArgs& a,
                                                int q, int cur, int64_t strip, int64_t w, bool own_lane,
                                                bool wv) {
    constexpr int R = ROWS - 2 * T;
    if (!own_lane || !wv) return;
    const PlanePartDesc& d = a.p[q];
    const int64_t y0 = strip * R;                      // owned row 0 of the tile
    const int64_t wp = a.wp;
    if (d.prev != -1 && y0 < T) {                      // top rows -> prev's bottom halo
        // prev == -2: the previous active rank's last partition (peer memory)
        uint32_t* base = d.prev >= 0 ? a.p[d.prev].S[cur ^ 1] : a.rprev_S[cur ^ 1];
        const int64_t prows = d.prev >= 0 ? a.p[d.prev].rows : a.rprev_rows;
        uint32_t* o = base + (prows + T + y0) * wp + w;
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (y0 + i < T && y0 + i < d.rows) o[i * wp] = sv[T + i];
    }
    if (d.next != -1 && y0 + R > d.rows - T) {         // bottom rows -> next's top halo
        uint32_t* o = (d.next >= 0 ? a.p[d.next].S[cur ^ 1] : a.rnext_S[cur ^ 1]) + w;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t y = y0 + i;
            if (y >= d.rows - T && y < d.rows) o[(y - d.rows + T) * wp] = sv[T + i];
        }
    }
}

// One pass of the multi-partition loop for one warp: the push-model activity
// and two-slot ring of plane_loop_pass_warp over the concatenated tile list.
// A live front also stamps across partition boundaries: a tile in a
// partition's first strip stamps the previous partition's last strip (and the
// one before it when that last strip has fewer than T rows — a front crosses
// it within one pass), a tile in the last strip (or in the second-to-last one
// when the last is short) the next partition's first strip.  Boundary strips
// whose neighbour is on another rank run every pass (its flags are not read).
template <int T, int ROWS>
__device__ __forceinline__ int plane_multi_pass_warp(const PlaneMultiArgs& a, int cur, int steps,
                                                     bool first, uint32_t stamp, int64_t gw,
                                                     int64_t nwarps, int lane, uint32_t* slots,
                                                     uint64_t* bars, uint32_t& phases) {
    constexpr int R = ROWS - 2 * T;
    constexpr int OW = 30;
    constexpr int BW = 36;
    constexpr uint32_t kBox = ROWS * BW * 4;
    const int64_t n_cb = a.n_cb;
    const bool own_lane = lane >= 1 && lane <= OW;
    if (a.total == 0) return -1;   // a rank without active partitions only joins the barriers
    uint32_t* __restrict__ act = a.act;
    const int64_t n_my = gw < a.total ? (a.total - gw + nwarps - 1) / nwarps : 0;
    auto part_of = [&](int64_t t) {
        int q = 0;
        while (q + 1 < a.np && t >= a.p[q + 1].tile0) ++q;
        return q;
    };
    auto short_last = [&](const PlanePartDesc& d) { return d.rows - (d.n_strips - 1) * R < T; };
    int64_t chunk = -1;
    uint32_t mask = 0;
    auto next_tile = [&]() -> int64_t {
        while (mask == 0) {
            ++chunk;
            if (chunk * 32 >= n_my) return -1;
            const int64_t i = chunk * 32 + lane;
            bool on = false;
            if (i < n_my) {
                const int64_t t = gw + i * nwarps;
                on = first || __ldcg(act + t) == stamp;
                if (!on) {
                    const PlanePartDesc& d = a.p[part_of(t)];
                    const int64_t strip = (t - d.tile0) / n_cb;
                    on = (d.prev == -2 && strip == 0) ||
                         (d.next == -2 && (strip == d.n_strips - 1 || (short_last(d) && strip == d.n_strips - 2)));
                }
            }
            mask = __ballot_sync(0xffffffffu, on);
        }
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        return gw + (chunk * 32 + b) * nwarps;
    };
    auto issue = [&](int64_t t, int s) {
        if (lane == 0) {
            const int q = part_of(t);
            const int64_t lt = t - a.p[q].tile0;
            const int64_t strip = lt / n_cb, cb = lt - strip * n_cb;
            const int x = (int)(cb * OW - 1) & ~3, y = (int)(strip * R);   // buffer row (hd = T)
            uint32_t* sb = slots + s * (2 * ROWS * BW);
            mbar_expect_tx(&bars[s], 2 * kBox);
            tma_load_2d(sb, &a.ts[q][cur], x, y, &bars[s]);
            tma_load_2d(sb + ROWS * BW, &a.tk[q], x, y, &bars[s]);
        }
    };
    int my_last = -1;
    int64_t t = next_tile();
    if (t >= 0) issue(t, 0);
    int64_t nxt = t >= 0 ? next_tile() : -1;
    if (nxt >= 0) issue(nxt, 1);
    int s = 0;
    while (t >= 0) {
        mbar_wait(&bars[s], (phases >> s) & 1u);
        phases ^= 1u << s;
        const int q = part_of(t);
        const PlanePartDesc& d = a.p[q];
        const int64_t lt = t - d.tile0;
        const uint32_t* sb = slots + s * (2 * ROWS * BW);
        const uint32_t* kb = sb + ROWS * BW;
        const int o = (int)((lt % n_cb) * OW - 1) & 3;
        uint32_t sv[ROWS], kv[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            sv[i] = sb[i * BW + o + lane];
            kv[i] = kb[i * BW + o + lane];
        }
        __syncwarp();                                  // slot s free: refill it
        const int64_t n2 = nxt >= 0 ? next_tile() : -1;
        if (n2 >= 0) issue(n2, s);
        const int64_t strip = lt / n_cb, cb = lt - strip * n_cb;
        const int64_t w = cb * OW - 1 + lane;
        const int tl = plane_steps<T, ROWS>(sv, kv, steps, own_lane, lane);
        my_last = max(my_last, tl);
        const bool wv = w >= 0 && w < a.wp;
        plane_store<T, ROWS>(sv, d.S[cur ^ 1], d.rows, a.wp, T, strip * R - T, w, own_lane, wv);
        plane_store_fwd<T, ROWS>(sv, a, q, cur, strip, w, own_lane, wv);
        if (tl >= 0) {
            const bool live = tl == steps - 1;
            int64_t target = -1;
            const int64_t c2 = cb + lane % 3 - 1;
            if (lane < 9) {   // the partition's own 3x3 neighbourhood (lane 4: the tile)
                const int64_t s2 = strip + lane / 3 - 1;
                if ((live || lane == 4) && s2 >= 0 && s2 < d.n_strips && c2 >= 0 && c2 < n_cb)
                    target = d.tile0 + s2 * n_cb + c2;
            } else if (live && lane < 18 && c2 >= 0 && c2 < n_cb) {
                if (lane < 15) {   // previous partition: last strip, and the one before a short one
                    if (strip == 0 && d.prev >= 0) {
                        const PlanePartDesc& pd = a.p[d.prev];
                        if (lane < 12) target = pd.tile0 + (pd.n_strips - 1) * n_cb + c2;
                        else if (short_last(pd) && pd.n_strips >= 2) target = pd.tile0 + (pd.n_strips - 2) * n_cb + c2;
                    }
                } else if (d.next >= 0 && (strip == d.n_strips - 1 || (short_last(d) && strip == d.n_strips - 2))) {
                    target = a.p[d.next].tile0 + c2;   // next partition: first strip
                }
            }
            if (target >= 0) act[target] = stamp + 1;
        }
        t = nxt;
        nxt = n2;
        s ^= 1;
    }
    return my_last;
}

template <int T, int ROWS>
__global__ void __launch_bounds__(256, 1) k_planes_multi(const __grid_constant__ PlaneMultiArgs a,
                                                      int64_t max_iters, int* __restrict__ flags,
                                                      int* __restrict__ state,
                                                      unsigned long long* __restrict__ prof) {
    constexpr int BW = 36;
    extern __shared__ __align__(128) uint32_t psm[];   // 8 x 2 warp slots, then 16 mbarriers
    uint64_t* bars = reinterpret_cast<uint64_t*>(psm + 8 * 2 * 2 * ROWS * BW);
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* slots = psm + wid * (2 * 2 * ROWS * BW);
    uint64_t* bar = &bars[2 * wid];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * 8 + wid;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    const bool xr = a.nranks > 1;
    int* own = xr ? a.xbar[a.rank] : nullptr;
    // arrivals of earlier runs (every rank ran the same passes: equal on all)
    const int epoch0 = xr && leader ? *((volatile int*)&own[1]) : 0;
    // act[total] = this run's stamp base (as in k_planes_loop)
    const uint32_t base = *((volatile uint32_t*)&a.act[a.total]);
    if (prof && leader) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        prof[0] = t;
    }
    uint32_t phases = 0;
    int64_t k0 = 0;
    int pass = 0;
    while (k0 < max_iters) {
        const int steps = (int)min((int64_t)T, max_iters - k0);
        if (leader) flags[(pass + 1) % 3] = -1;
        const int my_last = plane_multi_pass_warp<T, ROWS>(a, pass & 1, steps, pass == 0, base + (uint32_t)pass,
                                                           gw, nwarps, lane, slots, bar, phases);
        if (lane == 0 && my_last >= 0) atomicMax(&flags[pass % 3], (int)(k0 + my_last));
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xr) __threadfence_system();   // halo stores into peers before the rank barrier
        grid.sync();
        if (prof && leader && pass < 30) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[1 + pass] = t;
        }
        if (xr) {
            // rank barrier + all-reduce (max) of the last changing execution:
            // each leader publishes its value into every rank's slot, then
            // arrives on every rank's counter (release at system scope) and
            // waits for all arrivals of this pass on its own (acquire)
            if (leader) {
                const int slot = 4 + (pass % 3) * kXRanks;
                const int lv = *((volatile int*)&flags[pass % 3]);
                for (int r = 0; r < a.nranks; ++r)
                    asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(a.xbar[r] + slot + a.rank), "r"(lv)
                                 : "memory");
                __threadfence_system();
                for (int r = 0; r < a.nranks; ++r)
                    asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(a.xbar[r]) : "memory");
                const int target = epoch0 + (pass + 1) * a.nranks;
                unsigned long long t0;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                bool ok = true;
                for (;;) {
                    int cnt;
                    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(cnt) : "l"(own) : "memory");
                    if (cnt >= target) break;
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t - t0 > 10000000000ull) {   // 10 s: a rank is not running; abort
                        ok = false;
                        break;
                    }
                    __nanosleep(64);
                }
                int g = -1;
                for (int r = 0; r < a.nranks && ok; ++r) g = max(g, *((volatile int*)&own[slot + r]));
                flags[pass % 3] = ok ? g : INT_MIN;
            }
            grid.sync();
            asm volatile("fence.proxy.async.global;" ::: "memory");   // peers' halo rows, read by TMA
        }
        const int last = *((volatile int*)&flags[pass % 3]);
        if (last == INT_MIN) {   // cross-rank barrier timed out
            if (leader) {
                state[0] = (int)k0;
                state[1] = 0;
                state[2] = (pass & 1) ? 0 : 1;
                state[3] = -1;
                a.act[a.total] = base + (uint32_t)pass + 2;
                flags[0] = -1;   // ready for the next run (see k_planes_loop)
            }
            return;
        }
        if (last < k0 + steps - 1) {
            if (leader) {
                const int64_t last_global = last >= 0 ? last : k0 - 1;
                state[0] = (int)(last_global + 2);
                state[1] = 1;
                state[2] = (pass & 1) ? 0 : 1;
                state[3] = 0;
                if (xr) own[1] = epoch0 + (pass + 1) * a.nranks;
                a.act[a.total] = base + (uint32_t)pass + 2;
                flags[0] = -1;
            }
            return;
        }
        k0 += steps;
        ++pass;
    }
    if (leader) {
        state[0] = (int)max_iters;
        state[1] = 0;
        state[2] = pass == 0 ? 0 : (((pass - 1) & 1) ? 0 : 1);
        state[3] = 0;
        if (xr) own[1] = epoch0 + pass * a.nranks;
        a.act[a.total] = base + (uint32_t)pass + 2;
        flags[0] = -1;
    }
}


}  // namespace

int64_t hyst_tiles(int64_t rows, int64_t pitch) {
    return ((rows + kStencilRows - 1) / kStencilRows) *
           ((pitch / 16 + kStencilThreads - 1) / kStencilThreads);
}

cudaError_t hyst_step(const uint8_t* in, uint8_t* out, int64_t rows, int64_t pitch, int iter,
                      int* last_changed, const uint8_t* prev_flags, uint8_t* cur_flags,
                      int top_nbr, int bot_nbr, const Launch& L) {
    if (rows <= 0) return cudaSuccess;
    if (pitch % 16 != 0) return cudaErrorInvalidValue;
    static int occ = resident_ctas(k_hyst_step, kStencilThreads);
    int64_t strips = (rows + kStencilRows - 1) / kStencilRows;
    int64_t colblk = (pitch / 16 + kStencilThreads - 1) / kStencilThreads;
    ++g_launches;
    k_hyst_step<<<grid_for(strips * colblk, occ, L), kStencilThreads, 0, L.stream>>>(
        in, out, rows, pitch, iter, last_changed, strips, colblk, prev_flags, cur_flags, top_nbr,
        bot_nbr);
    return cudaGetLastError();
}
// rounded up to 4 words: the row pitch of a TMA tensor map is a multiple of 16 B
int64_t plane_words(int64_t W) { return (W + 127) / 128 * 4; }

// grid: x = resident CTAs split over the partitions (y), at least one each
static dim3 io_grid(const PlaneIO& io, int64_t per_row_items, int occ, const Launch& L) {
    int64_t tot = 0;
    for (int q = 0; q < io.np; ++q) tot += io.rows[q] * per_row_items;
    const unsigned gx = grid_for(tot, occ, L);
    return dim3(std::max(1u, gx / (unsigned)io.np), io.np);
}

cudaError_t planes_pack_io(const U8Prog& p, const PlaneIO& io, int64_t W, const Launch& L, int hd) {
    const int64_t wp = plane_words(W);
    if (io.np < 1 || io.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    for (int q = 0; q < io.np; ++q)
        if (io.rows[q] <= 0 || io.rows[q] * wp >= (1ll << 31)) return cudaErrorInvalidValue;
    const U8Const c = u8_consts(p);
    ++g_launches;
    const FastDiv WPd = make_fastdiv((uint32_t)wp);
#define MW_PACK(SEGV)                                                                       \
    {                                                                                       \
        static int occ = resident_ctas(k_planes_pack<SEGV>, 256);                           \
        k_planes_pack<SEGV><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(     \
            p, c, io, W, wp, WPd, hd);                                                      \
        return cudaGetLastError();                                                          \
    }
    if (p.n == 1 && p.kind[0] == U8_SEGMENT) {
        switch (c.lo_mode[0] * 4 + c.hi_mode[0]) {   // modes fixed at compile time
            case 0: MW_PACK(0)
            case 1: MW_PACK(1)
            case 2: MW_PACK(2)
            case 3: MW_PACK(3)
            case 5: MW_PACK(5)
            case 9: MW_PACK(9)
            case 10: MW_PACK(10)
            case 13: MW_PACK(13)
            case 14: MW_PACK(14)
            case 15: MW_PACK(15)
            default: break;
        }
    }
    MW_PACK(-1)
#undef MW_PACK
}

cudaError_t planes_pack(const U8Prog& p, const uint8_t* src, int64_t sp, int64_t rows, int64_t W,
                        uint32_t* S, uint32_t* K, const Launch& L, int hd) {
    if (rows <= 0) return cudaSuccess;
    PlaneIO io{};
    io.np = 1;
    io.sp = sp;
    io.src[0] = src;
    io.S0[0] = S;
    io.K[0] = K;
    io.rows[0] = rows;
    return planes_pack_io(p, io, W, L, hd);
}

cudaError_t planes_unpack_io(const U8Prog& p, const PlaneIO& io, const int* state, int64_t dp,
                             int64_t W, const Launch& L, int hd) {
    const int64_t wp = plane_words(W);
    if (io.np < 1 || io.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    bool dst_aligned = dp % 16 == 0, wide_ok = true;
    for (int q = 0; q < io.np; ++q) {
        if (io.rows[q] <= 0 || io.rows[q] * wp >= (1ll << 31)) return cudaErrorInvalidValue;
        dst_aligned &= (reinterpret_cast<uintptr_t>(io.dst[q]) & 15) == 0;
        wide_ok &= io.rows[q] * (wp / 128) < (1ll << 31);
    }
    const U8Const c = u8_consts(p);
    ++g_launches;
    if (p.n == 1 && p.kind[0] == U8_FINALIZE && wp % 128 == 0 && dst_aligned && wide_ok) {
        static int occ = resident_ctas(k_planes_unpack_fin_w, 256);
        // one warp per 128 plane words of a row
        dim3 g = io_grid(io, 1, occ, L);
        int64_t units = 0;
        for (int q = 0; q < io.np; ++q) units = std::max(units, io.rows[q] * (wp / 128));
        g.x = (unsigned)std::min<int64_t>(g.x, std::max<int64_t>(1, (units + 7) / 8));
        k_planes_unpack_fin_w<<<g, 256, 0, L.stream>>>(io, state, dp, wp,
                                                       make_fastdiv((uint32_t)(wp / 128)), hd);
    } else if (p.n == 1 && p.kind[0] == U8_FINALIZE) {
        static int occ = resident_ctas(k_planes_unpack<true>, 256);
        k_planes_unpack<true><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(
            p, c, io, state, dp, W, wp, make_fastdiv((uint32_t)wp), hd);
    } else {
        static int occ = resident_ctas(k_planes_unpack<false>, 256);
        k_planes_unpack<false><<<io_grid(io, (wp + 255) / 256, occ, L), 256, 0, L.stream>>>(
            p, c, io, state, dp, W, wp, make_fastdiv((uint32_t)wp), hd);
    }
    return cudaGetLastError();
}

cudaError_t planes_unpack(const U8Prog& p, const uint32_t* S0, const uint32_t* S1,
                          const uint32_t* K, const int* state, uint8_t* dst, int64_t dp,
                          int64_t rows, int64_t W, const Launch& L, int hd) {
    if (rows <= 0) return cudaSuccess;
    PlaneIO io{};
    io.np = 1;
    io.S0[0] = const_cast<uint32_t*>(S0);
    io.S1[0] = const_cast<uint32_t*>(S1);
    io.K[0] = const_cast<uint32_t*>(K);
    io.dst[0] = dst;
    io.rows[0] = rows;
    return planes_unpack_io(p, io, state, dp, W, L, hd);
}

int64_t planes_tiles(int64_t rows, int64_t W) {   // upper bound over the variants (R >= 8)
    return ((rows + 7) / 8) * ((plane_words(W) + 29) / 30);
}

// 2-D tensor map over a plane buffer of (rows + 2 hd) x wp words, box ROWS x 36
static bool plane_tmap(CUtensorMap* tm, const uint32_t* base, int64_t rows, int64_t wp, int box_rows,
                       int hd = 1) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = []() {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!enc) return false;
    // encoded maps are cached by (buffer, shape): the per-partition pass kernel
    // launches twice per partition and pass on the same scratch planes
    struct Key {
        const void* p;
        int64_t rows, wp;
        int box, hd;
        bool operator==(const Key& o) const {
            return p == o.p && rows == o.rows && wp == o.wp && box == o.box && hd == o.hd;
        }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.p) ^ (size_t)(k.rows * 1000003 + k.wp * 131 + k.box * 7 + k.hd);
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{base, rows, wp, box_rows, hd};
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *tm = it->second;
            return true;
        }
    }
    const cuuint64_t dims[2] = {(cuuint64_t)wp, (cuuint64_t)(rows + 2 * hd)};
    const cuuint64_t strides[1] = {(cuuint64_t)wp * 4};
    const cuuint32_t box[2] = {36, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    if (enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();   // bounded (freed scratch leaves stale keys)
    cache[key] = *tm;
    return true;
}

// MW_HYST_PROF=1: per-pass device timestamps of the loop kernel to stderr
static unsigned long long* hyst_prof_buf() {
    static unsigned long long* p = []() -> unsigned long long* {
        unsigned long long* q = nullptr;
        if (getenv("MW_HYST_PROF") && cudaMalloc(&q, 1024) != cudaSuccess) q = nullptr;
        return q;
    }();
    return p;
}
static void hyst_prof_print(const unsigned long long* prof, unsigned grid, int64_t tiles, cudaStream_t st) {
    unsigned long long h[128];
    cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "MW_HYST_PROF grid=%u tiles=%lld", grid, (long long)tiles);
    for (int i = 1; i < 32 && h[i]; ++i) fprintf(stderr, " %.1f", (h[i] - h[0]) / 1e3);
    fprintf(stderr, " us; tiles run / executions per pass:");
    for (int i = 0; i < 30 && h[64 + i]; ++i) fprintf(stderr, " %llu/%llu", h[64 + i], h[32 + i]);
    fprintf(stderr, "\n");
}

template <int T, int ROWS>
static cudaError_t planes_loop_t(uint32_t* S0, uint32_t* S1, const uint32_t* K, int64_t rows,
                                 int64_t wp, int64_t max_iters, int* flags, int* state,
                                 uint32_t* act, const Launch& L) {
    constexpr size_t smem = plane_loop_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_loop<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_loop<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    const int64_t tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    // cooperative: every CTA must be co-resident
    unsigned grid = grid_for((tiles + 7) / 8, occ, L);
    CUtensorMap ts0, ts1, tk;
    if (!plane_tmap(&ts0, S0, rows, wp, ROWS) || !plane_tmap(&ts1, S1, rows, wp, ROWS) ||
        !plane_tmap(&tk, K, rows, wp, ROWS))
        return cudaErrorInvalidValue;
    unsigned long long* prof = hyst_prof_buf();
    if (prof) cudaMemsetAsync(prof, 0, 1024, L.stream);
    int64_t r = rows, w = wp, mi = max_iters;
    void* args[] = {&ts0, &ts1, &tk, &S0, &S1, &r, &w, &mi, &flags, &state, &act, &prof};
    ++g_launches;
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_planes_loop<T, ROWS>, dim3(grid),
                                                dim3(256), args, smem, L.stream);
    if (prof && e == cudaSuccess) hyst_prof_print(prof, grid, tiles, L.stream);
    return e;
}

template <int T, int ROWS>
static cudaError_t planes_pass_t(const uint32_t* in, uint32_t* out, const uint32_t* K, int64_t rows,
                                 int64_t wp, int steps, int64_t k0, const uint8_t* fprev,
                                 uint8_t* fcur, int first, int top, int bot, int* last,
                                 const Launch& L) {
    constexpr size_t smem = plane_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_pass<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_pass<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    const int64_t tiles = ((rows + R - 1) / R) * ((wp + 29) / 30);
    CUtensorMap tin, tk;
    if (!plane_tmap(&tin, in, rows, wp, ROWS, T) || !plane_tmap(&tk, K, rows, wp, ROWS, T))
        return cudaErrorInvalidValue;
    ++g_launches;
    k_planes_pass<T, ROWS><<<grid_for((tiles + 7) / 8, occ, L), 256, smem, L.stream>>>(
        tin, tk, out, rows, wp, steps, k0, fprev, fcur, first, top, bot, last);
    return cudaGetLastError();
}

int planes_pass_depth(int T_pref, int64_t min_rows) {
    const int ts[] = {12, 8, 6, 4, 2, 1};
    for (int t : ts)
        if (t <= T_pref && t <= min_rows) return t;
    return 1;
}

cudaError_t planes_pass(const uint32_t* in, uint32_t* out, const uint32_t* K, int64_t rows,
                        int64_t W, int T, int steps, int64_t k0, const uint8_t* fprev,
                        uint8_t* fcur, int first, int top, int bot, int* last, const Launch& L) {
    const int64_t wp = plane_words(W);
    if (rows <= 0) return cudaSuccess;
    switch (T) {
        case 12: return planes_pass_t<12, 40>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 8: return planes_pass_t<8, 48>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 6: return planes_pass_t<6, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 4: return planes_pass_t<4, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        case 2: return planes_pass_t<2, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
        default: return planes_pass_t<1, 32>(in, out, K, rows, wp, steps, k0, fprev, fcur, first, top, bot, last, L);
    }
}

cudaError_t planes_loop(uint32_t* S0, uint32_t* S1, const uint32_t* K, int64_t rows, int64_t W,
                        int64_t max_iters, int* flags, int* state, uint32_t* act,
                        const Launch& L) {
    const int64_t wp = plane_words(W);
    const int T = L.tune[TUNE_HYST_T];
    const int ROWS = L.tune[TUNE_HYST_ROWS];
#define MW_PL(TT, RR) \
    if (T == TT && ROWS == RR) return planes_loop_t<TT, RR>(S0, S1, K, rows, wp, max_iters, flags, state, act, L)
    MW_PL(4, 32);
    MW_PL(6, 32);
    MW_PL(8, 32);
    MW_PL(8, 40);
    MW_PL(12, 40);
    MW_PL(8, 48);
    MW_PL(6, 48);
#undef MW_PL
    return planes_loop_t<8, 48>(S0, S1, K, rows, wp, max_iters, flags, state, act, L);
}

template <int T, int ROWS>
static cudaError_t planes_multi_t(const PlaneMultiHost& h, int64_t max_iters, int* flags, int* state,
                                  const Launch& L) {
    constexpr size_t smem = plane_loop_smem_bytes<ROWS>();
    static int occ = [] {
        cudaFuncSetAttribute(k_planes_multi<T, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return resident_ctas(k_planes_multi<T, ROWS>, 256, smem);
    }();
    constexpr int R = ROWS - 2 * T;
    static PlaneMultiArgs a;   // host staging of the (large) parameter block
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    a = PlaneMultiArgs{};
    a.np = h.np;
    a.wp = h.wp;
    a.n_cb = (h.wp + 29) / 30;
    a.rank = h.rank;
    a.nranks = h.nranks;
    if (h.nranks < 1 || h.nranks > kXRanks) return cudaErrorInvalidValue;
    for (int r = 0; r < h.nranks && h.nranks > 1; ++r) {
        if (!h.xbar[r]) return cudaErrorInvalidValue;
        a.xbar[r] = h.xbar[r];
    }
    a.rprev_S[0] = h.rprev_S[0];
    a.rprev_S[1] = h.rprev_S[1];
    a.rprev_rows = h.rprev_rows;
    a.rnext_S[0] = h.rnext_S[0];
    a.rnext_S[1] = h.rnext_S[1];
    int64_t tiles = 0;
    for (int q = 0; q < h.np; ++q) {
        PlanePartDesc& d = a.p[q];
        d.S[0] = h.S0[q];
        d.S[1] = h.S1[q];
        d.fl = h.fl[q];
        d.rows = h.rows[q];
        d.n_strips = (d.rows + R - 1) / R;
        d.nt = d.n_strips * a.n_cb;
        d.tile0 = tiles;
        tiles += d.nt;
        d.prev = q > 0 ? q - 1 : (h.remote_prev ? -2 : -1);
        d.next = q + 1 < h.np ? q + 1 : (h.remote_next ? -2 : -1);
        if (d.rows < T || 2 * d.nt > h.fl_bytes[q]) return cudaErrorInvalidValue;
        if (!plane_tmap(&a.ts[q][0], h.S0[q], d.rows, h.wp, ROWS, T) ||
            !plane_tmap(&a.ts[q][1], h.S1[q], d.rows, h.wp, ROWS, T) ||
            !plane_tmap(&a.tk[q], h.K[q], d.rows, h.wp, ROWS, T))
            return cudaErrorInvalidValue;
    }
    a.total = tiles;
    if (!h.act || h.act_words < tiles + 1) return cudaErrorInvalidValue;
    a.act = h.act;
    // loopback ranks share the GPU: each rank's cooperative grid takes its
    // share of the SMs so every rank's kernel is resident at the barriers
    const unsigned grid = std::max(1u, std::min(grid_for(std::max<int64_t>(1, (tiles + 7) / 8), occ, L),
                                                (unsigned)(sm_count() * occ / std::max(1, h.grid_div))));
    int64_t mi = max_iters;
    unsigned long long* prof = hyst_prof_buf();
    if (prof) cudaMemsetAsync(prof, 0, 1024, L.stream);
    void* args[] = {&a, &mi, &flags, &state, &prof};
    ++g_launches;
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_planes_multi<T, ROWS>, dim3(grid), dim3(256),
                                                args, smem, L.stream);
    if (prof && e == cudaSuccess) hyst_prof_print(prof, grid, tiles, L.stream);
    return e;
}

cudaError_t planes_multi(const PlaneMultiHost& h, int T, int64_t max_iters, int* flags, int* state,
                         const Launch& L) {
    if (h.np < (h.nranks > 1 ? 0 : 1) || h.np > kPlaneMaxParts) return cudaErrorInvalidValue;
    switch (T) {
        case 12: return planes_multi_t<12, 40>(h, max_iters, flags, state, L);
        case 8: return planes_multi_t<8, 48>(h, max_iters, flags, state, L);
        case 6: return planes_multi_t<6, 32>(h, max_iters, flags, state, L);
        case 4: return planes_multi_t<4, 32>(h, max_iters, flags, state, L);
        case 2: return planes_multi_t<2, 32>(h, max_iters, flags, state, L);
        default: return planes_multi_t<1, 32>(h, max_iters, flags, state, L);
    }
}

}  // namespace mwk
