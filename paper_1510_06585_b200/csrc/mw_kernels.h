// mw_kernels.h — internal launcher interface between the host runtime
// (exec.cpp, graph.cpp, profile.cpp) and the sm_100a kernels (chains.cu,
// planes.cu, nbody.cu, reduce.cu, fft.cu, kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace mwk {

constexpr int kMaxOps = 16;

// Launch geometry shared by every launcher: grid-stride kernels take a grid
// of min(work, SMs * resident CTAs); the slowdown injector divides that grid
// by `slow` (>= 1), which changes the speed but never the result.
// Tuning knobs (indices = MW_TUNE_* of marrow.h); every value gives
// bit-identical results, only speed changes.
enum TuneKnob : int {
    TUNE_RGBA_TMA = 0, TUNE_RGBA_UNROLL = 1, TUNE_HYST_PLANES = 2, TUNE_HYST_T = 3,
    TUNE_HYST_ROWS = 4, TUNE_NBODY_SPLIT = 5, TUNE_U8_TMA = 6, TUNE_HYST_FUSED = 7,
    TUNE_GRAPH_LANES = 8, TUNE_FFT_4STEP = 9, TUNE_COUNT = 10
};
void tune_defaults(int* out);                 // measured best on B200 (+ MW_* env overrides)
bool tune_valid(int knob, int value);
struct Launch {
    cudaStream_t stream;
    float slow;        // 1 = full speed
    const int* tune;   // TUNE_COUNT values
    // false: the launch reads nothing the stream's previous kernel wrote
    // (mw_ctx_set_run_pipelining), so it may issue its first loads before the
    // programmatic-dependent-launch wait (its stores still follow it)
    bool dep_wait = true;
    // per-ctx device scratch for launches that need one (the FFT dataflow
    // path's readiness counters: fft_work_bytes)
    void* work = nullptr;
    size_t work_bytes = 0;
};

// ------------------------------------------------------------ fused Map chains
// Saxpy chain: y <- fma(a_k, x, y) for k = 0..n-1, in place.
struct SaxpyProg {
    int n;
    float a[kMaxOps];
};
cudaError_t saxpy_chain(const SaxpyProg& p, const float* x, float* y, int64_t n, const Launch& L);

// RGBA8 chain: pointwise noise/solarize ops with every mirror
// folded into a source-column parity; key_mirror[k] says whether op k (a noise
// stage) runs at the mirrored column of the output pixel.
enum RgbaOpKind : int32_t { RGBA_NOISE = 0, RGBA_SOLARIZE = 1 };
struct RgbaProg {
    int n;
    int mirror;                     // odd number of mirrors in the chain
    int32_t kind[kMaxOps];
    uint32_t key[kMaxOps];          // NOISE: K = lowbias32(seed ^ 0x9E3779B9)
    int32_t param[kMaxOps];         // NOISE: scale S in [0,255]; SOLARIZE: T
    int32_t key_mirror[kMaxOps];
};
// rows x W pixels; row r of the partition is global row row0 + r.
cudaError_t rgba_chain(const RgbaProg& p, const uint8_t* src, uint8_t* dst, int64_t rows,
                       int64_t W, int64_t row0, const Launch& L);

// u8 chain: SEGMENT(lo,hi) / FINALIZE(128->0), rows of W bytes with pitches.
enum U8OpKind : int32_t { U8_SEGMENT = 0, U8_FINALIZE = 1 };
struct U8Prog {
    int n;
    int32_t kind[kMaxOps];
    int32_t lo[kMaxOps];
    int32_t hi[kMaxOps];
};
cudaError_t u8_chain(const U8Prog& p, const uint8_t* src, int64_t src_pitch, uint8_t* dst,
                     int64_t dst_pitch, int64_t rows, int64_t W, const Launch& L);

// ------------------------------------------------------------ hysteresis stencil
// One Jacobi step over `rows` interior rows.  in/out point at halo row -1 of
// buffers of (rows + 2) x pitch bytes (pitch % 16 == 0, pad columns zero).
// Any changed pixel does atomicMax(last_changed, iter).  Tiles whose 3x3
// neighbourhood did not change in the previous execution (prev_flags, one
// byte per tile; nullptr = all active) are skipped; cur_flags receives this
// execution's per-tile change flags.  top_nbr/bot_nbr: the partition has a
// neighbour whose halo row may change (its boundary tiles always run).
int64_t hyst_tiles(int64_t rows, int64_t pitch);
cudaError_t hyst_step(const uint8_t* in, uint8_t* out, int64_t rows, int64_t pitch, int iter,
                      int* last_changed, const uint8_t* prev_flags, uint8_t* cur_flags,
                      int top_nbr, int bot_nbr, const Launch& L);

// Bit-plane hysteresis (one partition per device): pack applies the chain
// before the loop (ending with the threshold) and writes the strong (S) and
// weak (K) planes of (rows + 2) x plane_words(W) words with zero halo rows
// (the caller zeroes rows 0 and rows+1 of S0, S1 and K); loop runs up to
// max_iters Jacobi executions in one cooperative kernel and writes
// state[0..2] = {executions E, converged, index of the final S buffer};
// unpack applies the chain after the loop and writes bytes.
int64_t plane_words(int64_t W);
// hd: halo rows above and below the interior in the plane buffers
cudaError_t planes_pack(const U8Prog& p, const uint8_t* src, int64_t sp, int64_t rows, int64_t W,
                        uint32_t* S, uint32_t* K, const Launch& L, int hd = 1);
// act: planes_tiles(rows, W) + 1 32-bit per-tile activity stamps (scratch;
// never needs clearing: the last word is the stamp base the kernel advances).
int64_t planes_tiles(int64_t rows, int64_t W);
cudaError_t planes_loop(uint32_t* S0, uint32_t* S1, const uint32_t* K, int64_t rows, int64_t W,
                        int64_t max_iters, int* flags, int* state, uint32_t* act,
                        const Launch& L);
cudaError_t planes_unpack(const U8Prog& p, const uint32_t* S0, const uint32_t* S1,
                          const uint32_t* K, const int* state, uint8_t* dst, int64_t dp,
                          int64_t rows, int64_t W, const Launch& L, int hd = 1);
// Up to 32 independent device copies in one launch.
struct CopyBatch {
    int n;
    const uint8_t* src[32];
    uint8_t* dst[32];
    int64_t bytes[32];
};
cudaError_t copy_batch(const CopyBatch& b, cudaStream_t s);
// Loopback transport (test-only, comm.cpp): dst[i] = op over r of srcs[r][i]
// in rank order; dt 0 int32 / 1 fp32 / 2 fp64, op 0 sum / 1 max / 2 min
// (the executor's max/min operands are never NaN: R28 partials use maxNum).
cudaError_t reduce_ranks(const void* const* srcs, int n, void* dst, size_t count, int dt, int op,
                         cudaStream_t s);
// Several partitions (or ranks): one pass of `steps` (<= T) executions over one
// partition whose buffers carry T halo rows; atomicMax(last, k0 + last changed).
int planes_pass_depth(int T_pref, int64_t min_rows);   // largest built T <= both
cudaError_t planes_pass(const uint32_t* in, uint32_t* out, const uint32_t* K, int64_t rows,
                        int64_t W, int T, int steps, int64_t k0, const uint8_t* fprev,
                        uint8_t* fcur, int first, int top, int bot, int* last, const Launch& L);

// The same over several partitions in ONE launch each (blockIdx.y = entry):
// entry q packs rows src[q] (pitch sp) into S0[q] / K[q], resp. unpacks
// (state[2] ? S1[q] : S0[q], K[q]) into dst[q] (pitch dp); rows[q] > 0.
constexpr int kPlaneMaxParts = 8;
struct PlaneIO {
    int np;
    int64_t sp;
    const uint8_t* src[kPlaneMaxParts];
    uint8_t* dst[kPlaneMaxParts];
    uint32_t* S0[kPlaneMaxParts];
    uint32_t* S1[kPlaneMaxParts];
    uint32_t* K[kPlaneMaxParts];
    int64_t rows[kPlaneMaxParts];
};
cudaError_t planes_pack_io(const U8Prog& p, const PlaneIO& io, int64_t W, const Launch& L, int hd);
cudaError_t planes_unpack_io(const U8Prog& p, const PlaneIO& io, const int* state, int64_t dp,
                             int64_t W, const Launch& L, int hd);
// Several partitions of one rank, the whole loop in ONE cooperative kernel
// (partitions in row order, every one with rows >= T; planes with T halo
// rows as for planes_pass; pack + the initial K / S0 halo exchange done by the
// caller).  Halos between consecutive partitions are exchanged inside the
// kernel (stores into the neighbour's halo rows).  state[0..2] as
// planes_loop (state[2]: index of the final buffer, S0 or S1, of every
// partition); flags: 3 ints of scratch.
struct PlanePartDesc {
    uint32_t* S[2];
    uint8_t* fl;                     // 2 x nt tile flags
    int64_t rows, n_strips, nt, tile0;
    int prev, next;                  // neighbouring partition in the table, -1 at the image edge
};
// Several RANKS (the cross-rank fused loop): prev / next == -2 marks a
// neighbour on another rank, whose plane buffers the kernel stores into
// directly (peer memory over NVLink; the same device for loopback ranks);
// after every pass the ranks meet in a barrier on the xbar blocks (one per
// rank: [0] arrival counter, [1] epoch = arrivals of earlier runs, [2]
// spare, [4 + 3 * kXRanks) the ranks' last-changed executions per pass
// slot), which also all-reduces the loop condition.
constexpr int kXRanks = 16;
constexpr int kXBlockInts = 4 + 3 * kXRanks;
struct PlaneMultiArgs {
    CUtensorMap ts[kPlaneMaxParts][2];
    CUtensorMap tk[kPlaneMaxParts];
    PlanePartDesc p[kPlaneMaxParts];
    int np;
    int64_t wp, n_cb, total;
    uint32_t* rprev_S[2];   // previous active rank's last partition (prev == -2)
    int64_t rprev_rows;
    uint32_t* rnext_S[2];   // next active rank's first partition (next == -2)
    int* xbar[kXRanks];     // every rank's barrier block
    int rank, nranks;       // nranks == 1: no cross-rank barrier
    uint32_t* act;          // total + 1 activity stamps (the last: the stamp base)
};
struct PlaneMultiHost {
    int np;                 // 0 allowed with nranks > 1 (the rank only joins the barriers)
    int64_t wp;
    uint32_t* S0[kPlaneMaxParts];
    uint32_t* S1[kPlaneMaxParts];
    const uint32_t* K[kPlaneMaxParts];
    uint8_t* fl[kPlaneMaxParts];
    int64_t fl_bytes[kPlaneMaxParts];
    int64_t rows[kPlaneMaxParts];
    bool remote_prev = false, remote_next = false;
    uint32_t* rprev_S[2]{};
    int64_t rprev_rows = 0;
    uint32_t* rnext_S[2]{};
    int* xbar[kXRanks]{};
    int rank = 0, nranks = 1;
    int grid_div = 1;       // loopback ranks share one GPU: each gets 1/grid_div of it
    uint32_t* act = nullptr;   // activity stamps over the concatenated tiles (scratch, never cleared)
    int64_t act_words = 0;     // >= tiles + 1
};
// state[3] = -1 when a cross-rank barrier timed out (10 s; the run aborted).
cudaError_t planes_multi(const PlaneMultiHost& h, int T, int64_t max_iters, int* flags, int* state,
                         const Launch& L);

// ------------------------------------------------------------ N-body
// Bodies [first, first+count) of N: direct-sum acceleration (fp32 per
// 256-source tile, fp64 across tiles and across the fixed source segments).
// mode 0: symplectic Euler step into pos_out/vel_out (same global indexing);
// mode 1: write a_i (fp32) to acc.  part: nbody_part_doubles(count) fp64 scratch.
int64_t nbody_part_doubles(int64_t count);
cudaError_t nbody(const float4* pos, const float4* vel, float4* pos_out, float4* vel_out,
                  float4* acc, int64_t first, int64_t count, int64_t N, float eps2, float dt,
                  int mode, double* part, const Launch& L);

// ------------------------------------------------------------ MapReduce
constexpr int kChunkLog2 = 16;      // canonical reduction chunk: 2^16 elements
// fp64 partial of every 2^16-element chunk of elements [first, first+count)
// (first % 2^16 == 0) into partials[chunk index]; y == nullptr: sum, else dot.
// x[0] (and y[0]) hold global element x0.
// op: MW_REDUCE_* (0 sum, 1 maxNum, 2 minNum).
// pre (dot only): the map stage is pipeline(saxpy chain, map_product): the
// terms are x * y' with y' = fma(pre.a[k], x, y) applied in order in fp32.
// term_map (reduction-stage term map, MW_TERM_*; -1 none) applies to every
// fp64 term before the fold.
cudaError_t reduce_chunks(const float* x, const float* y, int64_t x0, int64_t first,
                          int64_t count, int64_t total, double* partials, const Launch& L,
                          int op = 0, const SaxpyProg* pre = nullptr, int term_map = -1);
// Fixed-tree combine of nchunks partials into *result (one CTA), then the
// reduction-stage scalar maps (kind 0 sqrt, 1 scale by c) in order.
struct ScalarPost {
    int n;
    int kind[8];
    double c[8];
};
cudaError_t reduce_combine(const double* partials, int64_t nchunks, double* result,
                           cudaStream_t s, int op = 0, const ScalarPost* post = nullptr);
// partials[0..n) = the operator's identity (0, -inf, +inf)
cudaError_t reduce_fill_identity(double* partials, int64_t n, cudaStream_t s, int op);

// ------------------------------------------------------------ traits
cudaError_t fill_traits(int64_t* out, int64_t count, int64_t size, int64_t offset,
                        const Launch& L);

int sm_count();
void note_launch();   // count one launch of ours (mw_ctx_launch_count)

// ------------------------------------------------------------ FFT (NEXT-3)
// nfft transforms of N = 2^log2n complex64 points (interleaved re, im), a
// chain of nst stages (bit s of inv: inverse with 1/N); in may equal out.
bool fft_supported(int log2n);   // 13..16
// one-time per-device setup of the FFT twiddle table (mw_ctx_create)
cudaError_t fft_prepare(cudaStream_t s);
cudaError_t fft_chain(const float* in, float* out, int64_t nfft, int log2n, uint32_t inv, int nst,
                      const Launch& L);
// device scratch fft_chain needs in L.work for nfft transforms of 2^log2n
size_t fft_work_bytes(int64_t nfft, int log2n);
unsigned long long launch_count();  // kernels launched by this library

}  // namespace mwk
