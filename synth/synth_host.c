/*
 * synth_host.c — seeded synthetic input generators (host side).
 *
 * This module holds NO arithmetic of the method (no skeleton, no kernel
 * definition): only the counter-based SplitMix64 generator and the fixed
 * recipes that turn its outputs into the inputs of each workload
 * (restated in DESIGN.md "Input recipe").  Both the
 * oracle side (tests, cpu_baseline) and the CUDA side (tests, bench) draw
 * their inputs from this module; synth_dev.cu is the device twin of the same
 * generator.  Element i of every stream depends only on (seed, i), so any
 * partition of the domain regenerates exactly its own slice.
 *
 * SplitMix64 output i for seed s:
 *   z = s + (i+1)*0x9E3779B97F4A7C15
 *   z = (z ^ (z>>30)) * 0xBF58476D1CE4E5B9
 *   z = (z ^ (z>>27)) * 0x94D049BB133111EB
 *   z ^= z >> 31                               (all mod 2^64)
 * f32 U[-1,1) = (z>>40)*2^-23 - 1 ; f32 U[0,1) = (z>>40)*2^-24 (exact in fp32)
 * byte stream: element v is byte (v mod 8), little-endian, of z_{v/8}
 * RGBA8 pixel p: R,G,B = bytes 0..2 of z_p, A = 255
 * N-body body b: x,y,z = U[-1,1) of z_{3b+c}, w = mass; velocity 0
 */
#include <stdint.h>
#include <string.h>

static inline uint64_t sm64(uint64_t s, uint64_t i) {
    uint64_t z = s + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t synth_splitmix64(uint64_t seed, uint64_t i) { return sm64(seed, i); }

void synth_u64(uint64_t seed, uint64_t start, uint64_t count, uint64_t* out) {
    for (uint64_t k = 0; k < count; ++k) out[k] = sm64(seed, start + k);
}

void synth_f32_um11(uint64_t seed, uint64_t start, uint64_t count, float* out) {
    for (uint64_t k = 0; k < count; ++k)
        out[k] = (float)(sm64(seed, start + k) >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

void synth_f32_u01(uint64_t seed, uint64_t start, uint64_t count, float* out) {
    for (uint64_t k = 0; k < count; ++k)
        out[k] = (float)(sm64(seed, start + k) >> 40) * (1.0f / 16777216.0f);
}

void synth_u8_stream(uint64_t seed, uint64_t start, uint64_t count, uint8_t* out) {
    for (uint64_t k = 0; k < count; ++k) {
        uint64_t v = start + k;
        out[k] = (uint8_t)(sm64(seed, v >> 3) >> (8 * (v & 7)));
    }
}

void synth_rgba(uint64_t seed, uint64_t start_px, uint64_t count, uint8_t* out) {
    for (uint64_t k = 0; k < count; ++k) {
        uint64_t z = sm64(seed, start_px + k);
        out[4 * k + 0] = (uint8_t)(z);
        out[4 * k + 1] = (uint8_t)(z >> 8);
        out[4 * k + 2] = (uint8_t)(z >> 16);
        out[4 * k + 3] = 255;
    }
}

void synth_nbody(uint64_t seed, uint64_t start, uint64_t count, float mass,
                 float* pos4, float* vel4) {
    for (uint64_t k = 0; k < count; ++k) {
        uint64_t b = start + k;
        for (int c = 0; c < 3; ++c)
            pos4[4 * k + c] = (float)(sm64(seed, 3 * b + c) >> 40) * (1.0f / 8388608.0f) - 1.0f;
        pos4[4 * k + 3] = mass;
        if (vel4) memset(vel4 + 4 * k, 0, 4 * sizeof(float));
    }
}
