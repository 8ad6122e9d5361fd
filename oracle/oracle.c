/*
 * oracle.c — THE ORACLE: TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously correct single-threaded CPU implementation of the
 * built-in kernels of the hot path, written from the paper (/root/reference
 * PAPER.md, "P:n" = line n) and the readings listed in DESIGN.md §"Readings".
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path (paper_1510_06585_b200/),
 * and nothing here is called by the product.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see
 * __graft_entry__.build()).  Every fused multiply-add that the definition
 * wants is written explicitly (fmaf); everything else rounds per operation.
 *
 * Floating point: fp64 unless the paper fixes the precision (Saxpy is single
 * precision by P:740-741, so the oracle rounds exactly once to binary32 with
 * the C99 correctly rounded fmaf).
 *
 * Parity pins for every function live in tests/test_oracle_pins.py; the one
 * part with no pin to the paper itself is listed in DESIGN.md ("parity
 * unpinned": fidelity of noise/solarize/segmentation/N-body definitions to
 * the paper's unpublished OpenCL kernels — only our stated readings are
 * pinned).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Saxpy
 * P:740-742 (§4 "Saxpy ... computes a single-precision multiplication of a
 * constant with a vector added to another vector"): BLAS in-place
 * y_i <- a*x_i + y_i, binary32, one rounding (reading R8 in DESIGN.md).  */
void orc_saxpy(int64_t n, float a, const float* x, float* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = fmaf(a, x[i], y[i]);
}

/* ------------------------------------------------------------------ noise
 * P:725 names "Gaussian Noise" only.  Reading R1: per pixel at
 * global (y,x) with idx = y*W + x (u32), K = lowbias32(seed ^ 0x9E3779B9),
 * h = lowbias32(idx ^ K), for channel c in {R,G,B}:
 *   n_c = (popcount((h >> 10c) & 0x3FF) - 5) * S     (Binomial(10,1/2))
 *   out_c = min(255, max(0, in_c + n_c)),  out_A = in_A.                  */
uint32_t orc_lowbias32(uint32_t v) {
    v ^= v >> 16;
    v *= 0x7feb352du;
    v ^= v >> 15;
    v *= 0x846ca68bu;
    v ^= v >> 16;
    return v;
}

static int popcount10(uint32_t v) {
    int c = 0;
    for (int b = 0; b < 10; ++b) c += (v >> b) & 1u;
    return c;
}

/* y0: global row of in[0] (the Offset trait); 0 for the whole image. */
void orc_gauss_noise(int64_t H, int64_t W, const uint8_t* in, uint8_t* out,
                     uint32_t seed, int32_t S, int64_t y0) {
    uint32_t K = orc_lowbias32(seed ^ 0x9E3779B9u);
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            uint32_t idx = (uint32_t)((y0 + y) * W + x);
            uint32_t h = orc_lowbias32(idx ^ K);
            const uint8_t* p = in + 4 * (y * W + x);
            uint8_t* q = out + 4 * (y * W + x);
            for (int c = 0; c < 3; ++c) {
                int n = (popcount10((h >> (10 * c)) & 0x3FFu) - 5) * S;
                int v = (int)p[c] + n;
                if (v < 0) v = 0;
                if (v > 255) v = 255;
                q[c] = (uint8_t)v;
            }
            q[3] = p[3];
        }
    }
}

/* ------------------------------------------------------------------ solarize
 * P:725.  Reading R2: PIL convention, c in {R,G,B}: v >= T ? 255 - v : v;
 * alpha untouched.                                                         */
void orc_solarize(int64_t npx, const uint8_t* in, uint8_t* out, int32_t T) {
    for (int64_t i = 0; i < npx; ++i) {
        for (int c = 0; c < 3; ++c) {
            int v = in[4 * i + c];
            out[4 * i + c] = (uint8_t)(v >= T ? 255 - v : v);
        }
        out[4 * i + 3] = in[4 * i + 3];
    }
}

/* ------------------------------------------------------------------ mirror
 * P:725-726 ("independently applied to distinct lines of the image").
 * Reading R3: horizontal, out(y,x) = in(y, W-1-x), whole 4-byte pixel.     */
void orc_mirror(int64_t H, int64_t W, const uint8_t* in, uint8_t* out) {
    for (int64_t y = 0; y < H; ++y)
        for (int64_t x = 0; x < W; ++x)
            memcpy(out + 4 * (y * W + x), in + 4 * (y * W + (W - 1 - x)), 4);
}

/* ------------------------------------------------------------------ segmentation
 * P:743 ("changing its value to either white, gray or black").  Reading R6:
 * label(v) = 0 if v < lo; 128 if lo <= v < hi; 255 if v >= hi.  Also the
 * hysteresis threshold2d stage (reading R11).                              */
void orc_segment(int64_t n, const uint8_t* in, uint8_t* out, int32_t lo, int32_t hi) {
    for (int64_t i = 0; i < n; ++i) {
        int v = in[i];
        out[i] = (uint8_t)(v < lo ? 0 : (v < hi ? 128 : 255));
    }
}

/* ------------------------------------------------------------------ hysteresis
 * Not in the paper (BASELINE.json north_star); reading R11, the Fig. 1 shape
 * pipeline(threshold, loop(step), finalize).
 * step (Jacobi): L'(p) = 255 if L(p) = 128 and some 8-neighbour q inside the
 * image has L(q) = 255, else L(p).  Returns 1 if any pixel changed.         */
int orc_hyst_step(int64_t H, int64_t W, const uint8_t* L, uint8_t* Ln) {
    int changed = 0;
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            uint8_t v = L[y * W + x];
            uint8_t r = v;
            if (v == 128) {
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (dy == 0 && dx == 0) continue;
                        int64_t yy = y + dy, xx = x + dx;
                        if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                        if (L[yy * W + xx] == 255) r = 255;
                    }
            }
            Ln[y * W + x] = r;
            if (r != v) changed = 1;
        }
    }
    return changed;
}

/* finalize: weak (128) -> 0, everything else unchanged.                    */
void orc_hyst_finalize(int64_t n, const uint8_t* in, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)(in[i] == 128 ? 0 : in[i]);
}

/* Closed form of Loop(step) (R11): a multi-source breadth-first
 * search from every 255 pixel through 128 pixels (8-connectivity).  Weak
 * pixels at BFS level <= max_level are promoted to 255 (max_level < 0: no
 * limit, i.e. the fixed point).  Returns D = the largest level promoted
 * (0 if none); the while-loop then runs E = D + 1 body executions.
 * Returns -1 on allocation failure.                                         */
int64_t orc_hyst_bfs(int64_t H, int64_t W, const uint8_t* L, uint8_t* out, int64_t max_level) {
    int64_t n = H * W;
    memcpy(out, L, (size_t)n);
    uint32_t* q = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
    if (!q) return -1;
    int64_t head = 0, tail = 0;
    for (int64_t i = 0; i < n; ++i)
        if (L[i] == 255) q[tail++] = (uint32_t)i;
    int64_t level = 0, D = 0;
    while (head < tail && (max_level < 0 || level < max_level)) {
        int64_t end = tail;
        int promoted = 0;
        for (; head < end; ++head) {
            int64_t p = q[head], y = p / W, x = p % W;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                    int64_t j = yy * W + xx;
                    if (out[j] == 128) {
                        out[j] = 255;
                        q[tail++] = (uint32_t)j;
                        promoted = 1;
                    }
                }
        }
        ++level;
        if (promoted) D = level;
    }
    free(q);
    return D;
}

/* ------------------------------------------------------------------ N-body
 * P:734-737 (direct-sum "for each single body computes its interaction with
 * all the remainder").  Reading R12: a_i = sum_j m_j d_ij (|d_ij|^2+eps2)^-3/2,
 * d_ij = p_j - p_i, G = 1, j = i contributes exactly 0.  fp64, j in index
 * order.  Also returns C_i = sum_j |m_j d_ij (r^2+eps2)^-3/2| (conditioning).
 * targets == NULL means all bodies 0..nt-1.                                 */
void orc_nbody_accel(int64_t N, const float* pos4, float eps2, int64_t nt,
                     const int64_t* targets, double* acc3, double* cond_c) {
    for (int64_t t = 0; t < nt; ++t) {
        int64_t i = targets ? targets[t] : t;
        double xi = pos4[4 * i], yi = pos4[4 * i + 1], zi = pos4[4 * i + 2];
        double ax = 0, ay = 0, az = 0, C = 0;
        for (int64_t j = 0; j < N; ++j) {
            double dx = (double)pos4[4 * j] - xi;
            double dy = (double)pos4[4 * j + 1] - yi;
            double dz = (double)pos4[4 * j + 2] - zi;
            double d2 = dx * dx + dy * dy + dz * dz;
            double r2 = d2 + (double)eps2;
            double inv = 1.0 / sqrt(r2);
            double s = (double)pos4[4 * j + 3] * (inv * inv * inv);
            ax += dx * s;
            ay += dy * s;
            az += dz * s;
            C += fabs(s) * sqrt(d2);
        }
        acc3[3 * t] = ax;
        acc3[3 * t + 1] = ay;
        acc3[3 * t + 2] = az;
        if (cond_c) cond_c[t] = C;
    }
}

/* One step of symplectic Euler (reading R12): v' = v + a dt, p' = p + v' dt,
 * m unchanged; computed in fp64 and rounded once to fp32.                   */
void orc_nbody_step(int64_t N, const float* pos4, const float* vel4, float eps2, float dt,
                    float* pos_out, float* vel_out, double* acc3) {
    orc_nbody_accel(N, pos4, eps2, N, NULL, acc3, NULL);
    for (int64_t i = 0; i < N; ++i) {
        for (int c = 0; c < 3; ++c) {
            double v = (double)vel4[4 * i + c] + acc3[3 * i + c] * (double)dt;
            double p = (double)pos4[4 * i + c] + v * (double)dt;
            vel_out[4 * i + c] = (float)v;
            pos_out[4 * i + c] = (float)p;
        }
        vel_out[4 * i + 3] = vel4[4 * i + 3];
        pos_out[4 * i + 3] = pos4[4 * i + 3];
    }
}

/* ------------------------------------------------------------------ MapReduce
 * P:165, P:191-192, P:379 (map + reduction), merging function "+"
 * (P:705-707).  Reading R9: map per element, then a serial left fold in
 * Neumaier-compensated fp64; fp32 products x*y are exact in fp64.           */
static void neumaier_add(double* s, double* c, double x) {
    double t = *s + x;
    if (fabs(*s) >= fabs(x))
        *c += (*s - t) + x;
    else
        *c += (x - t) + *s;
    *s = t;
}

double orc_sum(int64_t n, const float* x) {
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) neumaier_add(&s, &c, (double)x[i]);
    return s + c;
}

double orc_dot(int64_t n, const float* x, const float* y) {
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) neumaier_add(&s, &c, (double)x[i] * (double)y[i]);
    return s + c;
}

/* The same serial fold continued over consecutive chunks: sc = {s, c} carries
 * the fold state, so folding chunks in order is identical to one fold over
 * their concatenation (used for inputs too large to hold at once).
 * y == NULL folds x (sum), else x*y (dot).  Result of the fold = s + c.     */
void orc_fold_chunk(int64_t n, const float* x, const float* y, double* sc) {
    for (int64_t i = 0; i < n; ++i)
        neumaier_add(&sc[0], &sc[1], y ? (double)x[i] * (double)y[i] : (double)x[i]);
}

/* Device reduction stage (NEXT-4; P:191 map_reduce(SCT map_stage, SCT
 * reduction_stage); reading R28): a serial left fold of the terms (x, or x*y
 * exact in fp64) with maxNum (is_min = 0) or minNum (is_min = 1): a NaN term
 * is ignored, acc starts at the identity -inf / +inf (the empty result).    */
double orc_fold_extreme(int64_t n, const float* x, const float* y, int is_min) {
    double acc = is_min ? INFINITY : -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        const double t = y ? (double)x[i] * (double)y[i] : (double)x[i];
        if (t != t) continue;                       /* NaN term: ignored */
        if (is_min ? (t < acc) : (t > acc)) acc = t;
    }
    return acc;
}

/* sum |terms| for the ill-conditioned tolerance branch. */
double orc_abs_sum(int64_t n, const float* x, const float* y) {
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i)
        neumaier_add(&s, &c, fabs(y ? (double)x[i] * (double)y[i] : (double)x[i]));
    return s + c;
}

/* Reduction-stage SCT with term maps (NEXT-4, R28): the
 * serial Neumaier fp64 fold of already formed fp64 terms (the same fold as
 * orc_sum / orc_dot, whose terms are formed from fp32 inputs).             */
double orc_sum_f64(int64_t n, const double* t) {
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) neumaier_add(&s, &c, t[i]);
    return s + c;
}
