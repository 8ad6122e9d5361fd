// profile.cpp — NEXT-2 / NEXT-4 control steps around the executor: the
// exhaustive knob sweep (mw_autotune), Alg. 1 profile building with the
// binary-search workload-distribution generator (mw_profile_build,
// P:511-589), the Fig. 5 decision process (mw_run_managed) and
// device classes with relative performance.
#include <cmath>
#include <cstdio>
#include <functional>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"

using namespace mwx;

extern "C" {

// ------------------------------------------------------------ profile building
// Arguments a run updates in place (Saxpy y, N-body state): profile
// building runs the tree many times and restores them afterwards.
struct Snapshots {
    mw_ctx* c;
    cudaStream_t s;
    std::vector<std::pair<const mw_arg*, void*>> snaps;
    static size_t bytes_of(const mw_arg& a) {
        int64_t n = a.mode == MW_COPY ? a.shape[0] : a.local_rows;
        return (size_t)(n * row_bytes(a));
    }
    mw_status take(const Node* r, const mw_arg* args, int nargs) {
        std::vector<int> inplace;
        const int ik = r->in_kind, ok = r->out_kind;
        if (ik == MW_VK_SAXPY && nargs == 2) inplace = {1};
        if (ik == MW_VK_NBODY && ok == MW_VK_NBODY && nargs == 2) inplace = {0, 1};
        for (int i : inplace) {
            void* p;
            MW_OK_OR_RETURN(scratch(c, "autotune_snap" + std::to_string(i), bytes_of(args[i]) + 16, s, &p));
            CUDA_OK(cudaMemcpyAsync(p, args[i].ptr, bytes_of(args[i]), cudaMemcpyDefault, s));
            snaps.push_back({&args[i], p});
        }
        return MW_OK;
    }
    mw_status restore() {
        for (auto& sn : snaps)
            CUDA_OK(cudaMemcpyAsync(sn.first->ptr, sn.second, bytes_of(*sn.first), cudaMemcpyDefault, s));
        return MW_OK;
    }
};

mw_status mw_autotune(mw_ctx* c, const mw_node* root, const mw_arg* args, int32_t nargs,
                      void* stream, int32_t reps, mw_kb* kb, int32_t* tune_out, double* best_ms) {
    if (!c || !root || (nargs > 0 && !args) || reps < 1) return fail(MW_E_INVALID_SPEC, "bad argument");
    if (c->destroyed) return fail(MW_E_STATE, "ctx was destroyed");
    CUDA_OK(cudaSetDevice(c->device));
    (void)cudaGetLastError();   // see mw_run
    const Node* r = reinterpret_cast<const Node*>(root);
    std::vector<Step> prog;
    MW_OK_OR_RETURN(mw::plan(r, &prog));
    bool has_rgba = false, has_stencil = false, has_nbody = false, has_u8 = false;
    for (const Step& st : prog) {
        has_u8 |= st.kind == StepKind::U8;
        has_rgba |= st.kind == StepKind::Rgba;
        has_stencil |= st.kind == StepKind::StencilFor || st.kind == StepKind::StencilWhile;
        has_nbody |= st.kind == StepKind::NbodyLoop || st.kind == StepKind::NbodyAccel;
    }
    using Tune = std::vector<int>;
    const Tune base(c->tune, c->tune + mwk::TUNE_COUNT);
    std::vector<Tune> cands{base};
    if (has_rgba) {
        for (int tma = 0; tma <= 9; ++tma)
            for (int un : {2, 4, 8}) {
                if (tma > 0 && un != base[mwk::TUNE_RGBA_UNROLL]) continue;
                Tune t = base;
                t[mwk::TUNE_RGBA_TMA] = tma;
                t[mwk::TUNE_RGBA_UNROLL] = un;
                cands.push_back(t);
            }
    }
    if (has_stencil) {
        const int pairs[7][2] = {{4, 32}, {6, 32}, {8, 32}, {8, 40}, {12, 40}, {6, 48}, {8, 48}};
        Tune t = base;
        t[mwk::TUNE_HYST_PLANES] = 0;
        cands.push_back(t);
        for (auto& pr : pairs) {
            Tune u = base;
            u[mwk::TUNE_HYST_PLANES] = 1;
            u[mwk::TUNE_HYST_T] = pr[0];
            u[mwk::TUNE_HYST_ROWS] = pr[1];
            cands.push_back(u);
        }
    }
    if (has_u8)
        for (int v : {0, 1}) {
            Tune t = base;
            t[mwk::TUNE_U8_TMA] = v;
            cands.push_back(t);
        }
    if (has_nbody)
        for (int sp : {0, 1}) {
            Tune t = base;
            t[mwk::TUNE_NBODY_SPLIT] = sp;
            cands.push_back(t);
        }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MW_OK_OR_RETURN(fifo_enter(c, s));
    Snapshots snap{c, s, {}};
    MW_OK_OR_RETURN(snap.take(r, args, nargs));
    auto restore = [&]() -> mw_status { return snap.restore(); };
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    mw_future f;
    f.ctx = c;
    double tmp[4] = {0, 0, 0, 0};
    f.res = tmp;   // host memory is fine: results are only written by D2H copies we sync on
    double best = 1e300;
    Tune best_t = base;
    mw_status st = MW_OK;
    for (const Tune& t : cands) {
        for (int k = 0; k < mwk::TUNE_COUNT; ++k) c->tune[k] = t[k];
        st = run(c, r, args, nargs, s, &f);   // warm-up (allocates scratch)
        if (st != MW_OK) break;
        CUDA_OK(cudaEventRecord(e0, s));
        for (int i = 0; i < reps && st == MW_OK; ++i) st = run(c, r, args, nargs, s, &f);
        if (st != MW_OK) break;
        CUDA_OK(cudaEventRecord(e1, s));
        CUDA_OK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        const double per = (double)ms / reps;
        if (per < best) {
            best = per;
            best_t = t;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int k = 0; k < mwk::TUNE_COUNT; ++k) c->tune[k] = best_t[k];
    MW_OK_OR_RETURN(restore());
    fifo_exit(c, s);
    CUDA_OK(cudaStreamSynchronize(s));
    if (st != MW_OK) return st;
    if (kb) {
        std::vector<int64_t> dims(args[0].shape, args[0].shape + args[0].ndim);
        MW_OK_OR_RETURN(mw_kb_store(kb, root, dims.data(), (int32_t)dims.size(), best_t.data(),
                                    c->dist.data(), c->P, best, MW_PROV_BUILT));
    }
    if (tune_out)
        for (int k = 0; k < mwk::TUNE_COUNT; ++k) tune_out[k] = best_t[k];
    if (best_ms) *best_ms = best;
    return MW_OK;
}


// ------------------------------------------------------------ device classes (NEXT-4)
mw_status mw_ctx_set_device_class(mw_ctx* c, int32_t part, int32_t cls, double rel_perf) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    if (part < 0 || part >= c->P || cls < 0 || !(rel_perf > 0.0) || !std::isfinite(rel_perf))
        return fail(MW_E_INVALID_SPEC, "bad partition, class or relative performance");
    c->cls[part] = cls;
    c->relperf[part] = rel_perf;
    // the static distribution is proportional to relative performance
    double tot = 0.0;
    for (double x : c->relperf) tot += x;
    for (int i = 0; i < c->P; ++i) c->dist[i] = c->relperf[i] / tot;
    return MW_OK;
}

void mw_profile_defaults(mw_profile_params* p) {
    if (!p) return;
    p->executions = 3;
    p->precision_ms = 0.0;
    p->max_dist_iters = 10;
}

}  // extern "C"

namespace {

// Per-partition compute times of the last run (this rank's view after the
// collective all-gather), for the workload distribution generator.
mw_status part_times(mw_ctx* c, std::vector<float>& ms) {
    ms.assign(c->P, 0.f);
    return mw_last_timings(c, ms.data(), c->P, nullptr);
}

// Workload distribution generator of Alg. 1: a binary search
// that moves load between two device types — class A (the class of the
// first partition) and the others.  The transferable share starts at 1,
// each iteration splits it evenly, binds one half to the type that
// performed better and keeps the other half transferable
// (transferableSize(n) = 1/2^n).  Inside a type the share follows the
// partitions' relative performance.  With one type it yields the
// relative-performance distribution once.
struct DistGen {
    const mw_ctx* c;
    int clsA = 0;
    bool two = false;
    double boundA = 0.0, boundB = 0.0, T = 1.0;
    int iter = 0;
    double lastA = 0.0;
    explicit DistGen(const mw_ctx* c_) : c(c_) {
        clsA = c->cls[0];
        for (int p = 0; p < c->P; ++p) two |= c->cls[p] != clsA;
    }
    bool done(int max_iters) const { return two ? iter >= max_iters : iter >= 1; }
    std::vector<double> next() {
        const double shareA = two ? boundA + T / 2 : 0.0;
        lastA = shareA;
        ++iter;
        std::vector<double> d(c->P, 0.0);
        double ra = 0.0, rb = 0.0;
        for (int p = 0; p < c->P; ++p) (c->cls[p] == clsA ? ra : rb) += c->relperf[p];
        for (int p = 0; p < c->P; ++p) {
            if (!two) d[p] = c->relperf[p] / ra;
            else if (c->cls[p] == clsA) d[p] = shareA * c->relperf[p] / ra;
            else d[p] = (1.0 - shareA) * c->relperf[p] / rb;
        }
        return d;
    }
    // per-type compute time of the proposal: the half goes to the faster type
    void feed(const std::vector<float>& ms) {
        if (!two) return;
        double ta = 0.0, tb = 0.0;
        for (int p = 0; p < c->P; ++p) (c->cls[p] == clsA ? ta : tb) = std::max(c->cls[p] == clsA ? ta : tb, (double)ms[p]);
        if (ta <= tb) boundA += T / 2;
        else boundB += T / 2;
        T /= 2;
    }
};

// One knob dimension of the configuration space: candidate settings, most
// likely first (P:555-565 ordering).
using Setting = std::vector<std::pair<int, int>>;
std::vector<std::vector<Setting>> config_dims(const mw_ctx* c, const std::vector<Step>& prog) {
    bool rgba = false, u8 = false, stencil = false, nbody = false, fft = false;
    for (const Step& st : prog) {
        rgba |= st.kind == StepKind::Rgba;
        u8 |= st.kind == StepKind::U8;
        stencil |= st.kind == StepKind::StencilFor || st.kind == StepKind::StencilWhile;
        nbody |= st.kind == StepKind::NbodyLoop || st.kind == StepKind::NbodyAccel;
        fft |= st.kind == StepKind::Fft;
    }
    std::vector<std::vector<Setting>> dims;
    auto ordered = [&](int knob, std::vector<int> vals) {
        std::vector<Setting> d{{{knob, c->tune[knob]}}};
        for (int v : vals)
            if (v != c->tune[knob]) d.push_back({{knob, v}});
        dims.push_back(d);
    };
    if (rgba) ordered(mwk::TUNE_RGBA_TMA, {1, 9, 5, 6, 3, 2, 4, 8, 7, 0});
    if (u8 && !stencil) ordered(mwk::TUNE_U8_TMA, {1, 0});
    if (stencil) {
        std::vector<Setting> d;
        d.push_back({{mwk::TUNE_HYST_PLANES, 1}, {mwk::TUNE_HYST_T, c->tune[mwk::TUNE_HYST_T]},
                     {mwk::TUNE_HYST_ROWS, c->tune[mwk::TUNE_HYST_ROWS]}});
        const int pairs[7][2] = {{8, 48}, {8, 40}, {6, 48}, {12, 40}, {6, 32}, {8, 32}, {4, 32}};
        for (auto& pr : pairs)
            if (pr[0] != c->tune[mwk::TUNE_HYST_T] || pr[1] != c->tune[mwk::TUNE_HYST_ROWS])
                d.push_back({{mwk::TUNE_HYST_PLANES, 1}, {mwk::TUNE_HYST_T, pr[0]}, {mwk::TUNE_HYST_ROWS, pr[1]}});
        d.push_back({{mwk::TUNE_HYST_PLANES, 0}});
        dims.push_back(d);
        if (c->ppr > 1) ordered(mwk::TUNE_HYST_FUSED, {1, 0});
    }
    if (nbody) ordered(mwk::TUNE_NBODY_SPLIT, {0, 1});
    if (fft) ordered(mwk::TUNE_FFT_4STEP, {1, 4, 2, 3, 0});
    return dims;
}

std::string wl_key(const mw_node* root, const mw_arg* args) {
    uint8_t id[32];
    mw_node_id(root, id);
    std::string k(reinterpret_cast<const char*>(id), 32);
    for (int d = 0; d < args[0].ndim; ++d) k += ":" + std::to_string(args[0].shape[d]);
    return k;
}

}  // namespace

extern "C" {

// Alg. 1 over the B200 configuration space: nested knob
// dimensions with the discard rule, the binary-search distribution
// generator innermost, store-if-better with the precision stop.
mw_status mw_profile_build(mw_ctx* c, const mw_node* root, const mw_arg* args, int32_t nargs,
                           void* stream, const mw_profile_params* pp, mw_kb* kb, int32_t* tune_out,
                           double* fractions_out, int32_t nfrac, double* best_ms, int32_t* runs_out) {
    if (!c || !root || (nargs > 0 && !args) || nargs < 1) return fail(MW_E_INVALID_SPEC, "bad argument");
    if (c->destroyed) return fail(MW_E_STATE, "ctx was destroyed");
    if (fractions_out && nfrac < c->P) return fail(MW_E_INVALID_SPEC, "fractions_out too small");
    mw_profile_params prm;
    mw_profile_defaults(&prm);
    if (pp) prm = *pp;
    if (prm.executions < 1 || prm.max_dist_iters < 1 || !(prm.precision_ms >= 0.0))
        return fail(MW_E_INVALID_SPEC, "bad profile parameters");
    CUDA_OK(cudaSetDevice(c->device));
    (void)cudaGetLastError();
    const Node* r = reinterpret_cast<const Node*>(root);
    std::vector<Step> prog;
    MW_OK_OR_RETURN(mw::plan(r, &prog));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MW_OK_OR_RETURN(fifo_enter(c, s));
    Snapshots snap{c, s, {}};
    MW_OK_OR_RETURN(snap.take(r, args, nargs));
    const bool mon0 = c->monitor;
    c->monitor = true;   // the generator needs per-partition times
    const std::vector<int> tune0(c->tune, c->tune + mwk::TUNE_COUNT);
    const std::vector<double> dist0 = c->dist;
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    mw_future f;
    f.ctx = c;
    double tmp[4] = {0, 0, 0, 0};
    f.res = tmp;
    double best = 1e300;
    std::vector<int> best_t = tune0;
    std::vector<double> best_d = dist0;
    int runs = 0;
    mw_status st = MW_OK;
    // exec_for_profile (step 13): warm-up + `executions` runs, mean time
    auto exec = [&](double* ms_out, std::vector<float>& parts) -> mw_status {
        MW_OK_OR_RETURN(run(c, r, args, nargs, s, &f));
        CUDA_OK(cudaEventRecord(e0, s));
        for (int i = 0; i < prm.executions; ++i) MW_OK_OR_RETURN(run(c, r, args, nargs, s, &f));
        CUDA_OK(cudaEventRecord(e1, s));
        CUDA_OK(cudaEventSynchronize(e1));
        runs += 1 + prm.executions;
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        *ms_out = (double)ms / prm.executions;
        MW_OK_OR_RETURN(part_times(c, parts));
        // Partitions sharing a device (ppr > 1) stand in for devices of their
        // own, which would run concurrently: the execution time of a
        // configuration is then the makespan, the longest partition's compute
        // time (the sum the shared stream takes is not what a multi-device
        // run would see).
        if (c->ppr > 1) *ms_out = (double)*std::max_element(parts.begin(), parts.end());
        return MW_OK;
    };
    // steps 9-20 for the current platform configuration: returns the best
    // time this configuration reached
    auto dist_search = [&]() -> double {
        DistGen gen(c);
        double here = 1e300;
        std::vector<float> parts;
        while (st == MW_OK && !gen.done(prm.max_dist_iters)) {
            const std::vector<double> d = gen.next();
            if (mw::check_distribution(d.data(), c->P) != MW_OK) break;
            c->dist = d;
            double t = 0.0;
            st = exec(&t, parts);
            if (st != MW_OK) break;
            here = std::min(here, t);
            if (getenv("MW_PROFILE_TRACE")) {
                fprintf(stderr, "profile: tune");
                for (int k = 0; k < mwk::TUNE_COUNT; ++k) fprintf(stderr, " %d", c->tune[k]);
                fprintf(stderr, " dist");
                for (double x : d) fprintf(stderr, " %.4f", x);
                fprintf(stderr, " ms %.4f parts", t);
                for (float x : parts) fprintf(stderr, " %.4f", x);
                fprintf(stderr, "\n");
            }
            gen.feed(parts);
            const double stored = best;
            if (t < stored) {   // store_profile (step 16)
                best = t;
                best_t.assign(c->tune, c->tune + mwk::TUNE_COUNT);
                best_d = d;
                if (stored - t < prm.precision_ms) break;   // step 17
            } else {
                break;
            }
        }
        return here;
    };
    const std::vector<std::vector<Setting>> dims = config_dims(c, prog);
    // nested configuration loops with the discard rule (steps 21, 23, 25):
    // a value that does not improve on the previous one discards the rest
    std::function<double(size_t)> search = [&](size_t level) -> double {
        if (level == dims.size()) return dist_search();
        double prev = 1e300, here = 1e300;
        for (const Setting& v : dims[level]) {
            if (st != MW_OK) break;
            for (auto& kv : v) c->tune[kv.first] = kv.second;
            const double t = search(level + 1);
            here = std::min(here, t);
            if (!(t < prev)) break;
            prev = t;
        }
        return here;
    };
    search(0);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int k = 0; k < mwk::TUNE_COUNT; ++k) c->tune[k] = best < 1e300 ? best_t[k] : tune0[k];
    c->dist = best < 1e300 ? best_d : dist0;
    c->monitor = mon0;
    MW_OK_OR_RETURN(snap.restore());
    fifo_exit(c, s);
    CUDA_OK(cudaStreamSynchronize(s));
    if (st != MW_OK) return st;
    if (kb) {
        std::vector<int64_t> dimsv(args[0].shape, args[0].shape + args[0].ndim);
        MW_OK_OR_RETURN(mw_kb_store(kb, root, dimsv.data(), (int32_t)dimsv.size(), c->tune, c->dist.data(), c->P,
                                    best, MW_PROV_BUILT));
    }
    if (tune_out)
        for (int k = 0; k < mwk::TUNE_COUNT; ++k) tune_out[k] = c->tune[k];
    if (fractions_out)
        for (int i = 0; i < c->P; ++i) fractions_out[i] = c->dist[i];
    if (best_ms) *best_ms = best;
    if (runs_out) *runs_out = runs;
    return MW_OK;
}

void mw_managed_defaults(mw_managed_params* p) {
    if (!p) return;
    mw_balance_defaults(&p->balance);
    p->build_profiles = 0;
    mw_profile_defaults(&p->profile);
}

// Persist the previous managed run's attained result (its wall time with
// the configuration it ran) with the process that produced it.
static mw_status managed_persist(mw_ctx* c) {
    if (!c->m_pending || !c->m_kb) return MW_OK;
    c->m_pending = false;
    float wall = 0.f;
    MW_OK_OR_RETURN(mw_last_timings(c, nullptr, 0, &wall));
    return mw_kb_store(c->m_kb, c->m_root, c->m_dims.data(), (int32_t)c->m_dims.size(), c->tune, c->dist.data(),
                       c->P, (double)wall, c->m_prov);
}

// Fig. 5: the decision process around a run request.
mw_status mw_run_managed(mw_ctx* c, mw_kb* kb, const mw_managed_params* mp, const mw_node* root,
                         const mw_arg* args, int32_t nargs, void* stream, mw_future** out,
                         int32_t* action) {
    if (!c || !kb || !root || !out || nargs < 1 || !args) return fail(MW_E_INVALID_SPEC, "NULL argument");
    if (c->destroyed) return fail(MW_E_STATE, "ctx was destroyed");
    mw_managed_params prm;
    mw_managed_defaults(&prm);
    if (mp) prm = *mp;
    if (!c->monitor) return fail(MW_E_STATE, "managed runs need monitoring (mw_ctx_set_monitoring)");
    const std::string key = wl_key(root, args);
    const std::vector<int64_t> dims(args[0].shape, args[0].shape + args[0].ndim);
    int act = MW_MANAGED_RECURRENT;
    if (c->m_pending && c->m_kb == kb && key == c->mkey) {
        // recurrent (SCT, workload): persist the last result, assess balance
        MW_OK_OR_RETURN(managed_persist(c));
        int32_t trig = 0;
        MW_OK_OR_RETURN(mw_rebalance(c, &prm.balance, &trig));
        int32_t found = 0, prov = 0;
        double ms = 0.0;
        MW_OK_OR_RETURN(mw_kb_find(kb, root, dims.data(), (int32_t)dims.size(), &found, &prov, &ms));
        if (prm.build_profiles && trig && !(found && prov == MW_PROV_BUILT)) {
            // "Build SCT profile": only once per (SCT, workload), when asked for
            MW_OK_OR_RETURN(mw_profile_build(c, root, args, nargs, stream, &prm.profile, kb, nullptr, nullptr, 0,
                                             nullptr, nullptr));
            c->bstate = mw_balance_state{};
            act = MW_MANAGED_BUILT;
            c->m_prov = MW_PROV_BUILT;
        } else if (trig) {
            act = MW_MANAGED_ADJUSTED;   // "Adjust workload distribution"
            c->m_prov = MW_PROV_BALANCED;
        }
    } else {
        // new (SCT, workload): "Derive work distribution" from the KB
        if (c->m_kb) MW_OK_OR_RETURN(managed_persist(c));
        int32_t scope = MW_KB_NONE;
        std::vector<int32_t> tune(c->tune, c->tune + mwk::TUNE_COUNT);
        std::vector<double> fr(c->P);
        MW_OK_OR_RETURN(mw_kb_lookup(kb, root, dims.data(), (int32_t)dims.size(), tune.data(), fr.data(), c->P,
                                     &scope));
        if (scope != MW_KB_NONE) {
            for (int k = 0; k < mwk::TUNE_COUNT; ++k)
                if (mwk::tune_valid(k, tune[k])) c->tune[k] = tune[k];
            if (mw::check_distribution(fr.data(), c->P) == MW_OK) c->dist = fr;
            act = scope == MW_KB_EXACT ? MW_MANAGED_FROM_KB : MW_MANAGED_DERIVED;
        } else {
            act = MW_MANAGED_NO_KNOWLEDGE;
        }
        c->m_prov = MW_PROV_DERIVED;
        c->bstate = mw_balance_state{};
        c->mkey = key;
        c->m_kb = kb;
        if (c->m_root != root) {   // keep the tree alive for the deferred KB store
            mw_node_retain(const_cast<mw_node*>(root));
            if (c->m_root) mw_node_release(const_cast<mw_node*>(c->m_root));
            c->m_root = root;
        }
        c->m_dims = dims;
    }
    MW_OK_OR_RETURN(mw_run(c, root, args, nargs, stream, out));
    c->m_pending = true;
    if (action) *action = act;
    return MW_OK;
}

mw_status mw_managed_flush(mw_ctx* c) {
    if (!c) return fail(MW_E_STATE, "NULL ctx");
    return managed_persist(c);
}

}  // extern "C"
