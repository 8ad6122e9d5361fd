// nbody.cu — the N-body Loop of Map step (R12): direct-sum
// softened accelerations in packed FP32x2 with fp64 across source tiles, then
// the symplectic Euler step; bound by the FP32 (FMA) pipe.
// Definitions follow DESIGN.md §Readings (R1-R12), citing PAPER.md lines.
#include "kcommon.cuh"

namespace mwk {
namespace {

// ------------------------------------------------------------ N-body
// a_i = sum_j m_j d_ij (|d_ij|^2 + eps2)^-3/2 (R12): fp32 inside each
// 256-source tile (global tile boundaries, so results do not depend on the
// partitioning), fp64 across tiles.  Four bodies per thread amortise the
// shared-memory broadcast loads; MUFU.RSQ for the inverse square root.
constexpr int kNbTile = 256;
constexpr int kNbPairs = 3;               // body pairs per thread (6 bodies; 2 and 4 measured slower)
constexpr int kNbPer = 2 * kNbPairs;
// The source range is cut into kNbSeg fixed tile-aligned segments: work
// items are (body block, segment), so the items of a partition fill the
// resident CTAs in many waves whatever its share — 2^20 bodies make 32784
// items for 296 resident CTAs (2 per SM: 111 waves), a 1/8 share 4128 (14
// waves, 99.6 % of the last one busy); with 3 segments a 1/2 share left its
// 4th wave half empty (1.75x instead of 2x the whole step's rate).  Each item
// writes its fp64 partial; k_nbody_fin sums the segments in order.  The split
// depends only on N, so results stay identical for every distribution of the
// bodies.
constexpr int kNbSeg = 48;

// Packed FP32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2): one instruction
// updates a pair of bodies; scalar operands are broadcast by ptxas.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& lo, float& hi) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float rsqrt_mufu(float x) {
    float r;  // MUFU.RSQ; x >= eps2 > 0 is never denormal, so .ftz is exact here
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Per interaction (for each body of a pair, in FP32x2 lanes):
//   d = p_j - p_i;  r2 = dx*dx + (dy*dy + (dz*dz + eps2));  inv = rsqrt(r2)
//   w = (m_j * inv) * (inv * inv);  f += d * w
// = 6 packed ops per coordinate triple + 6 more: 12 FP32x2 + 2 MUFU per pair.
template <bool SPLIT>
__global__ void __launch_bounds__(kNbTile) k_nbody(const float4* __restrict__ pos,
                                                   const float4* __restrict__ vel,
                                                   float4* __restrict__ pos_out,
                                                   float4* __restrict__ vel_out,
                                                   float4* __restrict__ acc_out, int64_t first,
                                                   int64_t count, int64_t N, float eps2, float dt,
                                                   int mode, double* __restrict__ part) {
    __shared__ float4 sp[kNbTile];
    __shared__ float2 bp[3][kNbPairs][kNbTile];
    const int64_t per_blk = (int64_t)kNbTile * kNbPer;
    const int64_t nblk = (count + per_blk - 1) / per_blk;
    const int64_t ntiles = (N + kNbTile - 1) / kNbTile;
    for (int64_t w = blockIdx.x; w < nblk * kNbSeg; w += gridDim.x) {
        const int64_t b = w / kNbSeg;
        const int seg = (int)(w - b * kNbSeg);
        const int64_t j0 = (ntiles * seg / kNbSeg) * kNbTile;
        const int64_t j1e = (ntiles * (seg + 1) / kNbSeg) * kNbTile;
        const int64_t j1 = j1e < N ? j1e : N;
        double ax[kNbPer], ay[kNbPer], az[kNbPer];
        // body positions live only as packed pairs (one aligned register pair each)
        f2_t px[kNbPairs], py[kNbPairs], pz[kNbPairs];
        // stage the pairs through shared memory so each lands in an aligned
        // register pair straight from an LDS.64 (no per-use re-pairing MOVs)
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kNbPairs; ++h) {
            float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f), b4 = a4;
            const int64_t la = b * per_blk + (2 * h) * kNbTile + threadIdx.x;
            const int64_t lb = la + kNbTile;
            if (la < count) a4 = pos[first + la];
            if (lb < count) b4 = pos[first + lb];
            bp[0][h][threadIdx.x] = make_float2(a4.x, b4.x);
            bp[1][h][threadIdx.x] = make_float2(a4.y, b4.y);
            bp[2][h][threadIdx.x] = make_float2(a4.z, b4.z);
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kNbPairs; ++h) {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(px[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[0][h][threadIdx.x])));
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(py[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[1][h][threadIdx.x])));
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(pz[h]) : "r"((unsigned)__cvta_generic_to_shared(&bp[2][h][threadIdx.x])));
        }
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) ax[q] = ay[q] = az[q] = 0.0;
        const f2_t e2 = f2_pack(eps2, eps2);
        for (int64_t jt = j0; jt < j1; jt += kNbTile) {
            __syncthreads();
            const int64_t j = jt + threadIdx.x;
            sp[threadIdx.x] = j < N ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass-0 pads
            __syncthreads();
            f2_t fx[kNbPairs], fy[kNbPairs], fz[kNbPairs];   // packed accumulators
            float gx[kNbPer], gy[kNbPer], gz[kNbPer];        // scalar accumulators (SPLIT)
#pragma unroll
            for (int h = 0; h < kNbPairs; ++h) fx[h] = fy[h] = fz[h] = 0ull;
#pragma unroll
            for (int q = 0; q < kNbPer; ++q) gx[q] = gy[q] = gz[q] = 0.f;
#pragma unroll 8
            for (int k = 0; k < kNbTile; ++k) {
                const float4 s4 = sp[k];
                const f2_t sx = f2_pack(s4.x, s4.x), sy = f2_pack(s4.y, s4.y),
                           sz = f2_pack(s4.z, s4.z), sw = f2_pack(s4.w, s4.w);
#pragma unroll
                for (int h = 0; h < kNbPairs; ++h) {
                    const f2_t dx = f2_sub(sx, px[h]), dy = f2_sub(sy, py[h]),
                               dz = f2_sub(sz, pz[h]);
                    const f2_t r2 = f2_fma(dx, dx, f2_fma(dy, dy, f2_fma(dz, dz, e2)));
                    float r0, r1;
                    f2_unpack(r2, r0, r1);
                    const f2_t inv = f2_pack(rsqrt_mufu(r0), rsqrt_mufu(r1));
                    if (SPLIT) {
                        // 8 packed ops on the FMA-heavy pipe, 8 scalar ops free to
                        // issue to the FMA-lite pipe (same roundings as the packed form)
                        const f2_t t = f2_mul(sw, inv), i2 = f2_mul(inv, inv);
                        float t0, t1, q0, q1, x0, x1, y0, y1, z0, z1;
                        f2_unpack(t, t0, t1);
                        f2_unpack(i2, q0, q1);
                        f2_unpack(dx, x0, x1);
                        f2_unpack(dy, y0, y1);
                        f2_unpack(dz, z0, z1);
                        const float w0 = t0 * q0, w1 = t1 * q1;
                        gx[2 * h] = __fmaf_rn(x0, w0, gx[2 * h]);
                        gx[2 * h + 1] = __fmaf_rn(x1, w1, gx[2 * h + 1]);
                        gy[2 * h] = __fmaf_rn(y0, w0, gy[2 * h]);
                        gy[2 * h + 1] = __fmaf_rn(y1, w1, gy[2 * h + 1]);
                        gz[2 * h] = __fmaf_rn(z0, w0, gz[2 * h]);
                        gz[2 * h + 1] = __fmaf_rn(z1, w1, gz[2 * h + 1]);
                    } else {
                        const f2_t w = f2_mul(f2_mul(sw, inv), f2_mul(inv, inv));
                        fx[h] = f2_fma(dx, w, fx[h]);
                        fy[h] = f2_fma(dy, w, fy[h]);
                        fz[h] = f2_fma(dz, w, fz[h]);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < kNbPairs; ++h) {
                float x0, x1, y0, y1, z0, z1;
                f2_unpack(fx[h], x0, x1);
                f2_unpack(fy[h], y0, y1);
                f2_unpack(fz[h], z0, z1);
                if (SPLIT) {
                    x0 = gx[2 * h]; x1 = gx[2 * h + 1];
                    y0 = gy[2 * h]; y1 = gy[2 * h + 1];
                    z0 = gz[2 * h]; z1 = gz[2 * h + 1];
                }
                ax[2 * h] += (double)x0; ax[2 * h + 1] += (double)x1;
                ay[2 * h] += (double)y0; ay[2 * h + 1] += (double)y1;
                az[2 * h] += (double)z0; az[2 * h + 1] += (double)z1;
            }
        }
#pragma unroll
        for (int q = 0; q < kNbPer; ++q) {
            const int64_t l = b * per_blk + q * kNbTile + threadIdx.x;
            if (l >= count) continue;
            double* o = part + (seg * count + l) * 3;
            o[0] = ax[q];
            o[1] = ay[q];
            o[2] = az[q];
        }
    }
}

// Sum the segment partials in order, then the epilogue: mode 1 writes a_i;
// mode 0 the symplectic Euler step (fp64 update, fp32 state).
__global__ void k_nbody_fin(const double* __restrict__ part, const float4* __restrict__ pos,
                            const float4* __restrict__ vel, float4* __restrict__ pos_out,
                            float4* __restrict__ vel_out, float4* __restrict__ acc_out,
                            int64_t first, int64_t count, float dt, int mode) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < count;
         l += (int64_t)gridDim.x * blockDim.x) {
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
        for (int sgi = 0; sgi < kNbSeg; ++sgi) {
            const double* o = part + (sgi * count + l) * 3;
            ax += o[0];
            ay += o[1];
            az += o[2];
        }
        const int64_t i = first + l;
        if (mode == 1) {
            acc_out[l] = make_float4((float)ax, (float)ay, (float)az, 0.f);
        } else {
            const float4 v = vel[i];
            const float4 pq = pos[i];
            const double d = (double)dt;
            const double vx = (double)v.x + ax * d, vy = (double)v.y + ay * d,
                         vz = (double)v.z + az * d;
            vel_out[i] = make_float4((float)vx, (float)vy, (float)vz, v.w);
            pos_out[i] = make_float4((float)((double)pq.x + vx * d),
                                     (float)((double)pq.y + vy * d),
                                     (float)((double)pq.z + vz * d), pq.w);
        }
    }
}


}  // namespace

int64_t nbody_part_doubles(int64_t count) { return (int64_t)kNbSeg * count * 3; }

cudaError_t nbody(const float4* pos, const float4* vel, float4* pos_out, float4* vel_out,
                  float4* acc, int64_t first, int64_t count, int64_t N, float eps2, float dt,
                  int mode, double* part, const Launch& L) {
    if (count <= 0) return cudaSuccess;
    // MW_NBODY_SPLIT: 1 = packed FP32x2 + scalar split across the FMA pipes (measured
    // slower on B200: 537 vs 519 ms per 2^20 step, so off by default)
    const int split = L.tune[TUNE_NBODY_SPLIT];
    const int64_t items = (count + kNbTile * kNbPer - 1) / (kNbTile * kNbPer) * kNbSeg;
    ++g_launches;
    if (split) {
        static int occ = resident_ctas(k_nbody<true>, kNbTile);
        k_nbody<true><<<grid_for(items, occ, L), kNbTile, 0, L.stream>>>(
            pos, vel, pos_out, vel_out, acc, first, count, N, eps2, dt, mode, part);
    } else {
        static int occ = resident_ctas(k_nbody<false>, kNbTile);
        k_nbody<false><<<grid_for(items, occ, L), kNbTile, 0, L.stream>>>(
            pos, vel, pos_out, vel_out, acc, first, count, N, eps2, dt, mode, part);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++g_launches;
    k_nbody_fin<<<grid_for((count + 255) / 256, 8, L), 256, 0, L.stream>>>(
        part, pos, vel, pos_out, vel_out, acc, first, count, dt, mode);
    return cudaGetLastError();
}


}  // namespace mwk
