// sct.cpp — skeleton computation tree construction and validation, fusion
// planner, partitioner and balancer (host, no device access).
//
// Paper: PAPER.md Table 1 constructors; P:217-224 bottom-up
// construction and LoopState; P:325-372 locality-aware decomposition and its
// constraint system; P:610-667 dynamic load balancing.  Readings: DESIGN.md.
#include "sct.h"

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <new>

namespace mw {

// ============================================================ errors
static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
mw_status fail(mw_status code, const std::string& msg) {
    t_err = msg;
    return code;
}
const char* last_error_cstr() { return t_err.c_str(); }

// ============================================================ tree helpers
void retain(Node* n) {
    if (n) __atomic_add_fetch(&n->refs, 1, __ATOMIC_RELAXED);
}
void release(Node* n) {
    if (!n) return;
    if (__atomic_sub_fetch(&n->refs, 1, __ATOMIC_ACQ_REL) == 0) {
        for (Node* k : n->kids) release(k);
        delete n->cache.load(std::memory_order_acquire);
        delete n;
    }
}

static const char* leaf_name(LeafKind k) {
    switch (k) {
        case LeafKind::Saxpy: return "saxpy";
        case LeafKind::GaussNoise: return "gauss_noise";
        case LeafKind::Solarize: return "solarize";
        case LeafKind::Mirror: return "mirror";
        case LeafKind::Segment: return "segment";
        case LeafKind::HystStep: return "hysteresis_step";
        case LeafKind::HystFinalize: return "hysteresis_finalize";
        case LeafKind::NbodyStep: return "nbody_step";
        case LeafKind::NbodyAccel: return "nbody_accel";
        case LeafKind::MapIdentity: return "map_identity";
        case LeafKind::MapProduct: return "map_product";
        case LeafKind::DebugTraits: return "debug_traits";
        case LeafKind::Fft: return "fft";
        case LeafKind::Reduce: return "reduce";
        case LeafKind::TermMap: return "term_map";
        case LeafKind::ScalarMap: return "scalar_map";
    }
    return "?";
}

std::string canonical(const Node* n) {
    char buf[256];
    switch (n->type) {
        case NodeType::Leaf:
            snprintf(buf, sizeof buf, "K(%s;%a;%a;%" PRId64 ";%" PRId64 ";%" PRId64 ")",
                     leaf_name(n->leaf), (double)n->fa, (double)n->fb, n->ia, n->ib, n->ic);
            return buf;
        case NodeType::Pipeline: {
            std::string s = "P(";
            for (const Node* k : n->kids) s += canonical(k) + ",";
            return s + ")";
        }
        case NodeType::Map: return "M(" + canonical(n->kids[0]) + ")";
        case NodeType::MapReduce:   // a user merge hashes by function address
            snprintf(buf, sizeof buf, "R(%d;%p;", n->merge_op, n->merge_op == MW_MERGE_USER ? n->fn : nullptr);
            return buf + canonical(n->kids[0]) +
                   (n->kids.size() > 1 ? "," + canonical(n->kids[1]) : std::string()) + ")";
        case NodeType::LoopHost:
            snprintf(buf, sizeof buf, "H(%" PRId64 ";%p;", n->n, n->fn);
            return buf + canonical(n->kids[0]) + ")";
        case NodeType::LoopFor:
            snprintf(buf, sizeof buf, "F(%" PRId64 ";", n->n);
            return buf + canonical(n->kids[0]) + ")";
        case NodeType::LoopWhile:
            snprintf(buf, sizeof buf, "W(%" PRId64 ";%d;", n->n, n->check_every);
            return buf + canonical(n->kids[0]) + ")";
    }
    return "";
}

void leaf_epu_nu(const Node* l, int64_t* epu, int64_t* nu) {
    if (l->leaf == LeafKind::DebugTraits) {
        *epu = l->ia;
        *nu = l->ib;
    } else {
        *epu = 1;  // image line / slab / element / body
        *nu = 1;   // B200 kernels bound-check tails (reading R5)
    }
}

std::vector<const Node*> leaves(const Node* n) {
    std::vector<const Node*> out;
    if (n->type == NodeType::Leaf) {
        out.push_back(n);
        return out;
    }
    for (const Node* k : n->kids) {
        auto v = leaves(k);
        out.insert(out.end(), v.begin(), v.end());
    }
    return out;
}

static bool compat(int a, int b) {
    auto u8 = [](int k) { return k == MW_VK_U8 || k == MW_VK_U8_2D; };
    // a saxpy value is the pair (x, y): two fp32 vectors, what map_product takes
    auto pair = [](int k) { return k == MW_VK_SAXPY || k == MW_VK_VEC2; };
    return a == b || (u8(a) && u8(b)) || (pair(a) && pair(b));
}
static bool has_2d(const Node* n) {
    if (n->type == NodeType::Leaf) return n->leaf == LeafKind::HystStep;
    for (const Node* k : n->kids)
        if (has_2d(k)) return true;
    return false;
}
static int norm2d(int kind, bool two_d) {
    return (two_d && kind == MW_VK_U8) ? MW_VK_U8_2D : kind;
}

// ============================================================ plan (fusion)
static bool is_chain(StepKind k) {
    return k == StepKind::Saxpy || k == StepKind::Rgba || k == StepKind::U8 || k == StepKind::Fft;
}
static void append_merged(std::vector<Step>& dst, const std::vector<Step>& src) {
    for (const Step& s : src) {
        if (!dst.empty()) {
            Step& b = dst.back();
            if (is_chain(s.kind) && b.kind == s.kind) {           // fuse the chain
                b.ops.insert(b.ops.end(), s.ops.begin(), s.ops.end());
                continue;
            }
            if (s.kind == StepKind::StencilFor && b.kind == StepKind::StencilFor) {
                b.n += s.n;
                continue;
            }
            if (s.kind == StepKind::NbodyLoop && b.kind == StepKind::NbodyLoop && b.dt == s.dt &&
                b.eps2 == s.eps2) {
                b.n += s.n;
                continue;
            }
        }
        dst.push_back(s);
    }
}

static constexpr int64_t kMaxChainOps = 1 << 16;

mw_status plan(const Node* n, std::vector<Step>* out) {
    out->clear();
    if (n->type == NodeType::Leaf) {
        Step s;
        ChainOp op{n->leaf, n->fa, n->ia, n->ib};
        switch (n->leaf) {
            case LeafKind::Saxpy: s.kind = StepKind::Saxpy; s.ops = {op}; break;
            case LeafKind::GaussNoise:
            case LeafKind::Solarize:
            case LeafKind::Mirror: s.kind = StepKind::Rgba; s.ops = {op}; break;
            case LeafKind::Segment:
            case LeafKind::HystFinalize: s.kind = StepKind::U8; s.ops = {op}; break;
            case LeafKind::HystStep: s.kind = StepKind::StencilFor; s.n = 1; break;
            case LeafKind::NbodyStep:
                s.kind = StepKind::NbodyLoop;
                s.n = 1;
                s.dt = n->fa;
                s.eps2 = n->fb;
                break;
            case LeafKind::NbodyAccel: s.kind = StepKind::NbodyAccel; s.eps2 = n->fb; break;
            case LeafKind::MapIdentity: s.kind = StepKind::MapStage; s.dot = false; break;
            case LeafKind::MapProduct: s.kind = StepKind::MapStage; s.dot = true; break;
            case LeafKind::Fft: s.kind = StepKind::Fft; s.ops = {op}; break;
            case LeafKind::Reduce:
            case LeafKind::TermMap:
            case LeafKind::ScalarMap:
                return fail(MW_E_INVALID_SPEC, "a reduction stage runs only inside mw_map_reduce_sct");
            case LeafKind::DebugTraits:
                s.kind = StepKind::Traits;
                s.epu = n->ia;
                s.nu = n->ib;
                s.strict = n->ic != 0;
                break;
        }
        out->push_back(s);
        return MW_OK;
    }
    std::vector<Step> a;
    switch (n->type) {
        case NodeType::Pipeline:
            for (const Node* k : n->kids) {
                mw_status st = plan(k, &a);
                if (st) return st;
                append_merged(*out, a);
            }
            return MW_OK;
        case NodeType::Map: return plan(n->kids[0], out);
        case NodeType::MapReduce: {
            mw_status st = plan(n->kids[0], &a);
            if (st) return st;
            // the map stage: map_identity / map_product, or a Map/Pipeline chain
            // of saxpy stages followed by map_product (fused: the chain's output
            // never leaves registers)
            std::vector<ChainOp> pre;
            if (a.size() == 2 && a[0].kind == StepKind::Saxpy && a[1].kind == StepKind::MapStage &&
                a[1].dot) {
                if ((int)a[0].ops.size() > 16)
                    return fail(MW_E_UNSUPPORTED, "map stage: saxpy chain longer than 16 stages");
                pre = a[0].ops;
                a.erase(a.begin());
            }
            if (a.size() != 1 || a[0].kind != StepKind::MapStage)
                return fail(MW_E_UNSUPPORTED,
                            "MapReduce map stage must be map_identity / map_product, or a saxpy "
                            "chain followed by map_product");
            Step s;
            s.kind = StepKind::Reduce;
            s.pre = pre;
            s.dot = a[0].dot;
            s.merge_op = n->merge_op;
            s.reduce_op = MW_REDUCE_SUM;
            if (n->kids.size() > 1) {
                // the reduction stage SCT: term maps, one reduce, scalar maps
                // (validated by mw_map_reduce_sct); composed term maps collapse
                // (abs o square = square o abs = square, abs o abs = abs, ...)
                for (const Node* l : leaves(n->kids[1])) {
                    if (l->leaf == LeafKind::TermMap) {
                        const int t = (int)l->ia;
                        s.term_map = s.term_map == MW_TERM_SQUARE || t == MW_TERM_SQUARE ? MW_TERM_SQUARE : t;
                    } else if (l->leaf == LeafKind::Reduce) {
                        s.reduce_op = (int32_t)l->ia;
                    } else if (l->leaf == LeafKind::ScalarMap) {
                        double c;
                        memcpy(&c, &l->ib, sizeof c);
                        s.post.push_back({(int32_t)l->ia, c});
                    }
                }
            }
            s.fn = n->fn;
            s.user = n->user;
            out->push_back(s);
            return MW_OK;
        }
        case NodeType::LoopFor: {
            mw_status st = plan(n->kids[0], &a);
            if (st) return st;
            if (a.size() == 1 && is_chain(a[0].kind)) {       // unrolled, fused
                if ((int64_t)a[0].ops.size() * n->n > kMaxChainOps)
                    return fail(MW_E_UNSUPPORTED, "loop over a chain unrolls to > 65536 stages");
                Step s;
                s.kind = a[0].kind;
                for (int64_t i = 0; i < n->n; ++i)
                    s.ops.insert(s.ops.end(), a[0].ops.begin(), a[0].ops.end());
                out->push_back(s);
                return MW_OK;
            }
            if (a.size() == 1 && (a[0].kind == StepKind::StencilFor || a[0].kind == StepKind::NbodyLoop)) {
                Step s = a[0];
                s.n = a[0].n * n->n;
                out->push_back(s);
                return MW_OK;
            }
            // any other body (mixed chains and stencils, nested while-loops, ...):
            // the loop is its body unrolled n times (P:376-378 with the state
            // carried between executions), adjacent chains / stencil steps merged
            if (n->n * (int64_t)a.size() > 4096)
                return fail(MW_E_UNSUPPORTED, "loop over a mixed body unrolls to > 4096 steps");
            for (int64_t i = 0; i < n->n; ++i) append_merged(*out, a);
            int64_t ops = 0;
            for (const Step& st : *out) ops += (int64_t)st.ops.size();
            if (ops > kMaxChainOps) return fail(MW_E_UNSUPPORTED, "loop unrolls to > 65536 chain stages");
            return MW_OK;
        }
        case NodeType::LoopWhile: {
            mw_status st = plan(n->kids[0], &a);
            if (st) return st;
            // the body is m >= 1 hysteresis steps (pipeline(step, step), loop_for(step, m),
            // ...): the only built-in kernel that reports change; the loop runs in steps
            // and reports body executions (a body changed iff one of its steps did)
            if (a.size() != 1 || a[0].kind != StepKind::StencilFor || a[0].n < 1)
                return fail(MW_E_UNSUPPORTED,
                            "LoopWhileChanged body must be hysteresis steps (the only built-in "
                            "kernel that reports change)");
            if (n->n > (int64_t{1} << 40) / a[0].n)
                return fail(MW_E_UNSUPPORTED, "while-loop step count overflows");
            Step s;
            s.kind = StepKind::StencilWhile;
            s.m = a[0].n;
            s.n = n->n * s.m;
            s.check_every = n->check_every;
            out->push_back(s);
            return MW_OK;
        }
        case NodeType::LoopHost:
            return fail(MW_E_UNSUPPORTED, "a host-condition loop (mw_loop_host) must be the root of the run");
        default: break;
    }
    return fail(MW_E_INVALID_SPEC, "unknown node type");
}

// ============================================================ granule / partition
static int64_t align_of(int kind) {
    switch (kind) {
        case MW_VK_SAXPY: return 4;          // 16-B float4 vectors
        case MW_VK_NBODY: return 256;        // one source tile of bodies
        case MW_VK_VEC1:
        case MW_VK_VEC2: return 1 << 16;     // canonical reduction chunk
        default: return 1;                   // one row / slab / element
    }
}

const NodeCache* plan_cached(const Node* root, mw_status* st) {
    Node* n = const_cast<Node*>(root);
    if (const NodeCache* c = n->cache.load(std::memory_order_acquire)) {
        *st = MW_OK;
        return c;
    }
    NodeCache* c = new NodeCache;
    *st = plan(root, &c->prog);
    if (*st != MW_OK) {   // errors are not cached (the message is per call)
        delete c;
        return nullptr;
    }
    c->granule = granule_of(root, &c->gst);
    c->strict = strict_of(root);
    NodeCache* expect = nullptr;
    if (!n->cache.compare_exchange_strong(expect, c, std::memory_order_acq_rel)) {
        delete c;   // another thread published first
        return expect;
    }
    return c;
}

int64_t granule_of(const Node* root, mw_status* st) {
    // a MapReduce root partitions by canonical reduction chunks whatever its
    // map stage's input kind (e.g. a saxpy chain fused into the map stage)
    int64_t g = root->out_kind == MW_VK_SCALAR ? align_of(MW_VK_VEC2) : align_of(root->in_kind);
    for (const Node* l : leaves(root)) {
        int64_t epu, nu;
        leaf_epu_nu(l, &epu, &nu);
        if (epu < 1 || nu < 1) {
            *st = fail(MW_E_INVALID_SPEC, "epu and nu must be >= 1");
            return 0;
        }
        if (epu % nu != 0) {   // P:365-366 first constraint family
            *st = fail(MW_E_EPU_NU, "epu mod nu != 0 (P:365-366): epu=" + std::to_string(epu) +
                                        " nu=" + std::to_string(nu));
            return 0;
        }
        g = std::lcm(g, epu / nu);
    }
    *st = MW_OK;
    return g;
}

bool strict_of(const Node* root) {
    for (const Node* l : leaves(root))
        if (l->leaf == LeafKind::DebugTraits && l->ic) return true;
    return false;
}

mw_status check_distribution(const double* d, int k) {
    if (!d || k < 1) return fail(MW_E_INVALID_SPEC, "empty distribution");
    double s = 0.0;
    bool pos = false;
    for (int i = 0; i < k; ++i) {
        if (!(d[i] >= 0.0)) return fail(MW_E_INVALID_SPEC, "negative or NaN fraction");
        if (d[i] > 0.0) pos = true;
        s += d[i];
    }
    if (!pos) return fail(MW_E_INVALID_SPEC, "no positive fraction");
    if (std::fabs(s - 1.0) > 1e-9)
        return fail(MW_E_INVALID_SPEC, "fractions must sum to 1 (+-1e-9)");
    return MW_OK;
}

// Largest remainder (reading R13) — keep in step with DESIGN.md.
mw_status partition_plan(int64_t L, int64_t g, const double* d, int k, bool strict,
                         int64_t* off, int64_t* len) {
    if (L < 0 || g < 1) return fail(MW_E_INVALID_SPEC, "bad domain length or granule");
    mw_status st = check_distribution(d, k);
    if (st) return st;
    const int64_t U = L / g, tail = L - U * g;
    if (strict && tail)
        return fail(MW_E_INFEASIBLE_PARTITION,
                    "strict partitioning: domain " + std::to_string(L) + " mod granule " +
                        std::to_string(g) + " != 0 (P:368)");
    std::vector<double> raw(k);
    std::vector<int64_t> base(k);
    int64_t sum = 0;
    for (int i = 0; i < k; ++i) {
        raw[i] = d[i] * (double)U;
        base[i] = (int64_t)std::floor(raw[i]);
        sum += base[i];
    }
    int64_t left = U - sum;
    std::vector<int> cand;
    for (int i = 0; i < k; ++i)
        if (d[i] > 0.0) cand.push_back(i);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
        double fa = raw[a] - (double)base[a], fb = raw[b] - (double)base[b];
        if (fa != fb) return fa > fb;
        if (d[a] != d[b]) return d[a] > d[b];
        return a < b;
    });
    for (int64_t j = 0; j < left; ++j) base[cand[j % (int64_t)cand.size()]] += 1;
    for (int64_t j = (int64_t)cand.size() - 1; left < 0; --j) {
        int i = cand[((j % (int64_t)cand.size()) + cand.size()) % cand.size()];
        if (base[i] > 0) {
            base[i] -= 1;
            left += 1;
        }
    }
    int last = cand.back();
    for (int i : cand) last = std::max(last, i);
    int64_t acc = 0;
    for (int i = 0; i < k; ++i) {
        int64_t n = base[i] * g + (i == last ? tail : 0);
        off[i] = acc;
        len[i] = n;
        acc += n;
    }
    return MW_OK;
}

// ============================================================ balancer (R15-R17)
mw_status balance_step(const mw_balance_params& p, mw_balance_state& s, const float* ms,
                       const int64_t* len, const double* cur, int n, double* next, int* trig) {
    if (n < 1 || !ms || !len || !cur || !next) return fail(MW_E_INVALID_SPEC, "bad balance args");
    if (!(p.weight > 0.0 && p.weight < 1.0) || !(p.c_factor > 0.0))
        return fail(MW_E_INVALID_SPEC, "weight must be in (0,1) and c_factor > 0");
    // dev = min/max of per-partition times over partitions with work
    double lo = 0, hi = 0;
    int act = 0;
    for (int i = 0; i < n; ++i) {
        if (len[i] <= 0) continue;
        double t = (double)ms[i];
        if (act == 0) lo = hi = t;
        lo = std::min(lo, t);
        hi = std::max(hi, t);
        ++act;
    }
    double dev = (act <= 1 || hi <= 0.0) ? 1.0 : lo / hi;
    int unb = (dev / p.c_factor < p.max_dev) ? 1 : 0;
    s.lbt = (double)unb * p.weight + s.lbt * (1.0 - p.weight);
    s.runs += 1;
    for (int i = 0; i < n; ++i) next[i] = cur[i];
    *trig = 0;
    if (s.active && !unb) {
        s.active = 0;
        s.lbt = 0.0;
        s.abs_t = 0.0;
        s.abs_last_dir = 0;
        s.abs_count = 0;
        return MW_OK;
    }
    if (!s.active && s.lbt < p.trigger) return MW_OK;
    if (p.mode == MW_BALANCE_PROPORTIONAL) {
        std::vector<double> r(n, 0.0);
        double tot = 0.0;
        for (int i = 0; i < n; ++i) {
            if (len[i] > 0) {
                double t = (double)ms[i];
                r[i] = (double)len[i] / (t > 0.0 ? t : 1e-30);
                tot += r[i];
            }
        }
        for (int i = 0; i < n; ++i) next[i] = r[i] / tot;
        s.lbt = 0.0;
        *trig = 1;
        return MW_OK;
    }
    if (p.mode != MW_BALANCE_ABS) return fail(MW_E_INVALID_SPEC, "unknown balance mode");
    if (n != 2) return fail(MW_E_INVALID_SPEC, "ABS mode needs exactly two partitions");
    s.active = 1;
    int d = ((double)ms[0] < (double)ms[1]) ? 1 : -1;
    if (s.abs_t == 0.0) s.abs_t = 0.125;
    if (d == s.abs_last_dir) {
        if (s.abs_count > 2) {
            s.abs_t = std::min(2.0 * s.abs_t, 1.0);
            s.abs_count = 0;
        }
        s.abs_count += 1;
    } else {
        if (s.abs_last_dir != 0) s.abs_t = s.abs_t / 2.0;
        s.abs_count = 1;
    }
    s.abs_last_dir = d;
    double s0 = cur[0] + (double)d * s.abs_t;
    s0 = s0 < 0.0 ? 0.0 : (s0 > 1.0 ? 1.0 : s0);
    s.lbt = 0.0;
    next[0] = s0;
    next[1] = 1.0 - s0;
    *trig = 1;
    return MW_OK;
}

// ============================================================ SHA-256 (FIPS 180-4)
void sha256(const void* data, size_t len, uint8_t out[32]) {
    static const uint32_t K[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
        0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
        0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
        0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
        0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
        0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
        0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
        0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
        0xc67178f2};
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    std::vector<uint8_t> m((const uint8_t*)data, (const uint8_t*)data + len);
    m.push_back(0x80);
    while (m.size() % 64 != 56) m.push_back(0);
    uint64_t bits = (uint64_t)len * 8;
    for (int i = 7; i >= 0; --i) m.push_back((uint8_t)(bits >> (8 * i)));
    auto rotr = [](uint32_t x, int r) { return (x >> r) | (x << (32 - r)); };
    for (size_t off = 0; off < m.size(); off += 64) {
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t)m[off + 4 * i] << 24 | (uint32_t)m[off + 4 * i + 1] << 16 |
                   (uint32_t)m[off + 4 * i + 2] << 8 | m[off + 4 * i + 3];
        for (int i = 16; i < 64; ++i) {
            uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
            uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int i = 0; i < 64; ++i) {
            uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
            uint32_t ch = (e & f) ^ (~e & g);
            uint32_t t1 = hh + S1 + ch + K[i] + w[i];
            uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
            uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            uint32_t t2 = S0 + mj;
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
}

}  // namespace mw

// ============================================================ C-ABI: nodes
using mw::fail;
using mw::LeafKind;
using mw::Node;
using mw::NodeType;

#define MW_TRY(...)                                                    \
    try {                                                              \
        __VA_ARGS__                                                    \
    } catch (const std::bad_alloc&) {                                  \
        return fail(MW_E_OOM, "host allocation failed");               \
    } catch (...) {                                                    \
        return fail(MW_E_INVALID_SPEC, "internal error");              \
    }

static mw_status make_leaf(LeafKind k, int in_kind, int out_kind, mw_node** out,
                           float fa = 0, float fb = 0, int64_t ia = 0, int64_t ib = 0,
                           int64_t ic = 0) {
    if (!out) return fail(MW_E_INVALID_SPEC, "out is NULL");
    MW_TRY({
        Node* n = new Node;
        n->type = NodeType::Leaf;
        n->leaf = k;
        n->fa = fa;
        n->fb = fb;
        n->ia = ia;
        n->ib = ib;
        n->ic = ic;
        n->in_kind = in_kind;
        n->out_kind = out_kind;
        *out = reinterpret_cast<mw_node*>(n);
        return MW_OK;
    })
}

extern "C" {

mw_status mw_kernel_saxpy(float a, mw_node** out) {
    return make_leaf(LeafKind::Saxpy, MW_VK_SAXPY, MW_VK_SAXPY, out, a);
}
mw_status mw_kernel_gauss_noise(uint32_t seed, int32_t scale, mw_node** out) {
    if (scale < 0 || scale > 255) return fail(MW_E_INVALID_SPEC, "noise scale must be in [0,255]");
    return make_leaf(LeafKind::GaussNoise, MW_VK_RGBA, MW_VK_RGBA, out, 0, 0, seed, scale);
}
mw_status mw_kernel_solarize(int32_t threshold, mw_node** out) {
    if (threshold < 0 || threshold > 256)
        return fail(MW_E_INVALID_SPEC, "solarize threshold must be in [0,256]");
    return make_leaf(LeafKind::Solarize, MW_VK_RGBA, MW_VK_RGBA, out, 0, 0, threshold);
}
mw_status mw_kernel_mirror(mw_node** out) {
    return make_leaf(LeafKind::Mirror, MW_VK_RGBA, MW_VK_RGBA, out);
}
mw_status mw_kernel_segment(int32_t lo, int32_t hi, mw_node** out) {
    if (lo < 0 || hi > 256 || lo > hi)
        return fail(MW_E_INVALID_SPEC, "segment needs 0 <= lo <= hi <= 256");
    return make_leaf(LeafKind::Segment, MW_VK_U8, MW_VK_U8, out, 0, 0, lo, hi);
}
mw_status mw_kernel_hysteresis_step(mw_node** out) {
    return make_leaf(LeafKind::HystStep, MW_VK_U8_2D, MW_VK_U8_2D, out);
}
mw_status mw_kernel_hysteresis_finalize(mw_node** out) {
    return make_leaf(LeafKind::HystFinalize, MW_VK_U8, MW_VK_U8, out);
}
mw_status mw_kernel_nbody_step(float dt, float eps2, mw_node** out) {
    if (!(eps2 > 0.f) || !std::isfinite(dt))
        return fail(MW_E_INVALID_SPEC, "nbody needs eps2 > 0 and finite dt");
    return make_leaf(LeafKind::NbodyStep, MW_VK_NBODY, MW_VK_NBODY, out, dt, eps2);
}
mw_status mw_kernel_nbody_accel(float eps2, mw_node** out) {
    if (!(eps2 > 0.f)) return fail(MW_E_INVALID_SPEC, "nbody needs eps2 > 0");
    return make_leaf(LeafKind::NbodyAccel, MW_VK_NBODY, MW_VK_ACCEL, out, 0, eps2);
}
mw_status mw_kernel_map_identity(mw_node** out) {
    return make_leaf(LeafKind::MapIdentity, MW_VK_VEC1, MW_VK_TERMS, out);
}
mw_status mw_kernel_map_product(mw_node** out) {
    return make_leaf(LeafKind::MapProduct, MW_VK_VEC2, MW_VK_TERMS, out);
}
mw_status mw_kernel_fft(int32_t log2n, int32_t inverse, mw_node** out) {
    if (log2n < 13 || log2n > 16)
        return fail(MW_E_INVALID_SPEC, "fft: log2n must be in 13..16 (N = 8192..65536 points)");
    if (inverse != 0 && inverse != 1) return fail(MW_E_INVALID_SPEC, "fft: inverse must be 0 or 1");
    return make_leaf(LeafKind::Fft, MW_VK_CPLX, MW_VK_CPLX, out, 0, 0, log2n, inverse);
}
mw_status mw_kernel_debug_traits(int64_t epu, int64_t nu, int32_t strict, mw_node** out) {
    if (epu < 1 || nu < 1) return fail(MW_E_INVALID_SPEC, "epu and nu must be >= 1");
    if (epu % nu != 0)
        return fail(MW_E_EPU_NU, "epu mod nu != 0 (P:365-366, S:127)");
    return make_leaf(LeafKind::DebugTraits, MW_VK_TRAITS, MW_VK_TRAITS, out, 0, 0, epu, nu,
                     strict ? 1 : 0);
}

static mw_status make_comp(NodeType t, mw_node* const* kids, int n, mw_node** out, int64_t cnt,
                           int32_t ce, int32_t op) {
    if (!out) return fail(MW_E_INVALID_SPEC, "out is NULL");
    for (int i = 0; i < n; ++i)
        if (!kids[i]) return fail(MW_E_INVALID_SPEC, "NULL child node");
    std::vector<Node*> ks;
    for (int i = 0; i < n; ++i) ks.push_back(reinterpret_cast<Node*>(kids[i]));
    bool two_d = false;
    for (Node* k : ks) two_d |= mw::has_2d(k);
    int in_kind = mw::norm2d(ks[0]->in_kind, two_d), out_kind = mw::norm2d(ks.back()->out_kind, two_d);
    switch (t) {
        case NodeType::Pipeline:
            if (n < 2) return fail(MW_E_INVALID_SPEC, "Pipeline needs >= 2 stages (S:68)");
            for (int i = 0; i + 1 < n; ++i)
                if (!mw::compat(ks[i]->out_kind, ks[i + 1]->in_kind))
                    return fail(MW_E_INVALID_SPEC, "pipeline stage " + std::to_string(i) +
                                                       " output kind does not feed stage " +
                                                       std::to_string(i + 1));
            break;
        case NodeType::MapReduce:
            if (ks[0]->out_kind != MW_VK_TERMS)
                return fail(MW_E_INVALID_SPEC, "MapReduce map stage must produce terms");
            if (op < MW_MERGE_ADD || op > MW_MERGE_USER)
                return fail(MW_E_INVALID_SPEC, "unknown merging function");
            out_kind = MW_VK_SCALAR;
            break;
        case NodeType::LoopFor:
        case NodeType::LoopWhile:
        case NodeType::LoopHost:
            if (!mw::compat(ks[0]->in_kind, ks[0]->out_kind))
                return fail(MW_E_INVALID_SPEC, "loop body must preserve its value kind");
            if (cnt < 0) return fail(MW_E_INVALID_SPEC, "loop count must be >= 0");
            if (t == NodeType::LoopWhile && ce < 1)
                return fail(MW_E_INVALID_SPEC, "check_every must be >= 1");
            break;
        default: break;
    }
    MW_TRY({
        Node* nd = new Node;
        nd->type = t;
        nd->kids = ks;
        for (Node* k : ks) mw::retain(k);
        nd->n = cnt;
        nd->check_every = ce;
        nd->merge_op = op;
        nd->in_kind = in_kind;
        nd->out_kind = out_kind;
        *out = reinterpret_cast<mw_node*>(nd);
        return MW_OK;
    })
}

mw_status mw_pipeline(mw_node* const* stages, int32_t n, mw_node** out) {
    if (!stages || n < 2) return fail(MW_E_INVALID_SPEC, "Pipeline needs >= 2 stages (S:68)");
    return make_comp(NodeType::Pipeline, stages, n, out, 0, 1, 0);
}
mw_status mw_map(mw_node* tree, mw_node** out) {
    return make_comp(NodeType::Map, &tree, 1, out, 0, 1, 0);
}
mw_status mw_map_reduce(mw_node* map_stage, int32_t merge_op, mw_node** out) {
    if (merge_op == MW_MERGE_USER)
        return fail(MW_E_INVALID_SPEC, "MW_MERGE_USER needs mw_map_reduce_user (a function)");
    return make_comp(NodeType::MapReduce, &map_stage, 1, out, 0, 1, merge_op);
}
mw_status mw_kernel_reduce(int32_t op, mw_node** out) {
    if (op < MW_REDUCE_SUM || op > MW_REDUCE_MIN) return fail(MW_E_INVALID_SPEC, "unknown reduction operator");
    return make_leaf(LeafKind::Reduce, MW_VK_TERMS, MW_VK_SCALAR, out, 0, 0, op);
}
mw_status mw_kernel_term_map(int32_t kind, mw_node** out) {
    if (kind != MW_TERM_ABS && kind != MW_TERM_SQUARE) return fail(MW_E_INVALID_SPEC, "unknown term map");
    return make_leaf(LeafKind::TermMap, MW_VK_TERMS, MW_VK_TERMS, out, 0, 0, kind);
}
mw_status mw_kernel_scalar_map(int32_t kind, double c, mw_node** out) {
    if (kind != MW_SCALAR_SQRT && kind != MW_SCALAR_SCALE) return fail(MW_E_INVALID_SPEC, "unknown scalar map");
    if (kind == MW_SCALAR_SCALE && !std::isfinite(c)) return fail(MW_E_INVALID_SPEC, "scale must be finite");
    if (kind == MW_SCALAR_SQRT) c = 0.0;
    int64_t bits;
    memcpy(&bits, &c, sizeof bits);
    return make_leaf(LeafKind::ScalarMap, MW_VK_SCALAR, MW_VK_SCALAR, out, 0, 0, kind, bits);
}
mw_status mw_map_reduce_sct(mw_node* map_stage, mw_node* reduction_stage, mw_node** out) {
    if (!reduction_stage) return fail(MW_E_INVALID_SPEC, "NULL reduction stage");
    const Node* r = reinterpret_cast<const Node*>(reduction_stage);
    // the reduction stage SCT: a reduce leaf, or a pipeline of term maps, ONE
    // reduce leaf and scalar maps (the kinds enforce the order)
    int nred = 0;
    bool ok = r->in_kind == MW_VK_TERMS && r->out_kind == MW_VK_SCALAR &&
              (r->type == NodeType::Leaf || r->type == NodeType::Pipeline);
    if (ok && r->type == NodeType::Pipeline)
        for (const Node* k : r->kids) ok &= k->type == NodeType::Leaf;
    for (const Node* l : leaves(r)) {
        nred += l->leaf == LeafKind::Reduce;
        ok &= l->leaf == LeafKind::Reduce || l->leaf == LeafKind::TermMap || l->leaf == LeafKind::ScalarMap;
    }
    if (!ok || nred != 1)
        return fail(MW_E_INVALID_SPEC, "the reduction stage must be a reduce leaf or a pipeline of term "
                                       "maps, one reduce leaf and scalar maps");
    mw_node* kids[2] = {map_stage, reduction_stage};
    return make_comp(NodeType::MapReduce, kids, 2, out, 0, 1, MW_MERGE_ADD);
}
mw_status mw_map_reduce_user(mw_node* map_stage, mw_merge_fn fn, void* user, mw_node** out) {
    if (!fn) return fail(MW_E_INVALID_SPEC, "NULL merging function");
    mw_status st = make_comp(NodeType::MapReduce, &map_stage, 1, out, 0, 1, MW_MERGE_USER);
    if (st) return st;
    Node* nd = reinterpret_cast<Node*>(*out);
    nd->fn = reinterpret_cast<void*>(fn);
    nd->user = user;
    return MW_OK;
}
mw_status mw_loop_host(mw_node* body, int64_t max_iters, mw_loop_cond_fn cond, void* user,
                       mw_node** out) {
    if (!cond) return fail(MW_E_INVALID_SPEC, "NULL loop condition");
    mw_status st = make_comp(NodeType::LoopHost, &body, 1, out, max_iters, 1, 0);
    if (st) return st;
    Node* nd = reinterpret_cast<Node*>(*out);
    nd->fn = reinterpret_cast<void*>(cond);
    nd->user = user;
    return MW_OK;
}
mw_status mw_loop_for(mw_node* body, int64_t n, mw_node** out) {
    return make_comp(NodeType::LoopFor, &body, 1, out, n, 1, 0);
}
mw_status mw_loop_while_changed(mw_node* body, int64_t max_iters, int32_t check_every,
                                mw_node** out) {
    return make_comp(NodeType::LoopWhile, &body, 1, out, max_iters, check_every, 0);
}
void mw_node_retain(mw_node* n) { mw::retain(reinterpret_cast<Node*>(n)); }
void mw_node_release(mw_node* n) { mw::release(reinterpret_cast<Node*>(n)); }

mw_status mw_node_id(const mw_node* n, uint8_t out[32]) {
    if (!n || !out) return fail(MW_E_INVALID_SPEC, "NULL argument");
    MW_TRY({
        std::string s = mw::canonical(reinterpret_cast<const Node*>(n));
        mw::sha256(s.data(), s.size(), out);
        return MW_OK;
    })
}
mw_status mw_node_signature(const mw_node* n, int32_t* in_kind, int32_t* out_kind) {
    if (!n) return fail(MW_E_INVALID_SPEC, "NULL node");
    const Node* nd = reinterpret_cast<const Node*>(n);
    if (in_kind) *in_kind = nd->in_kind;
    if (out_kind) *out_kind = nd->out_kind;
    return MW_OK;
}

static int64_t count_leaves(const Node* n) {
    if (n->type == NodeType::Leaf) return 1;
    int64_t c = 0;
    for (const Node* k : n->kids) c += count_leaves(k);
    return c;
}
static int64_t count_while(const Node* n) {
    int64_t c = (n->type == NodeType::LoopWhile || n->type == NodeType::LoopHost) ? 1 : 0;
    for (const Node* k : n->kids) c += count_while(k);
    return c;
}
// lb / wb: pre-order index of the first leaf / while-node occurrence in n.
static mw_status exec_order(const Node* n, int64_t lb, int64_t wb, const int64_t* wc,
                            std::vector<int32_t>& out) {
    if (out.size() > (size_t)1 << 28) return fail(MW_E_INVALID_SPEC, "execution order too long");
    switch (n->type) {
        case NodeType::Leaf: out.push_back((int32_t)lb); return MW_OK;
        case NodeType::LoopFor:
            for (int64_t i = 0; i < n->n; ++i) {
                mw_status st = exec_order(n->kids[0], lb, wb, wc, out);
                if (st) return st;
            }
            return MW_OK;
        case NodeType::LoopWhile:
        case NodeType::LoopHost:
            for (int64_t i = 0; i < wc[wb]; ++i) {
                mw_status st = exec_order(n->kids[0], lb, wb + 1, wc, out);
                if (st) return st;
            }
            return MW_OK;
        default:
            for (const Node* k : n->kids) {
                mw_status st = exec_order(k, lb, wb, wc, out);
                if (st) return st;
                lb += count_leaves(k);
                wb += count_while(k);
            }
            return MW_OK;
    }
}

mw_status mw_kernel_execution_order(const mw_node* root, const int64_t* while_counts,
                                    int32_t n_counts, int32_t* out_ids, int64_t* inout_len) {
    if (!root || !inout_len) return fail(MW_E_INVALID_SPEC, "NULL argument");
    MW_TRY({
        const Node* r = reinterpret_cast<const Node*>(root);
        int64_t need = count_while(r);
        if (n_counts < need || (need > 0 && !while_counts))
            return fail(MW_E_MISSING_ITERATION_COUNT,
                        "a LoopWhileChanged node has no iteration count (S:78)");
        for (int64_t i = 0; i < need; ++i)
            if (while_counts[i] < 0) return fail(MW_E_INVALID_SPEC, "negative iteration count");
        std::vector<int32_t> out;
        mw_status st = exec_order(r, 0, 0, while_counts, out);
        if (st) return st;
        if ((int64_t)out.size() > *inout_len || (!out_ids && !out.empty())) {
            *inout_len = (int64_t)out.size();
            return fail(MW_E_INVALID_SPEC, "output capacity too small");
        }
        for (size_t i = 0; i < out.size(); ++i) out_ids[i] = out[i];
        *inout_len = (int64_t)out.size();
        return MW_OK;
    })
}

mw_status mw_granule(const mw_node* root, int64_t* out) {
    if (!root || !out) return fail(MW_E_INVALID_SPEC, "NULL argument");
    MW_TRY({
        mw_status st;
        int64_t g = mw::granule_of(reinterpret_cast<const Node*>(root), &st);
        if (st) return st;
        *out = g;
        return MW_OK;
    })
}

mw_status mw_partition_plan(int64_t L, int64_t g, const double* fractions, int32_t k,
                            int32_t strict, int64_t* offsets, int64_t* lengths) {
    if (!offsets || !lengths) return fail(MW_E_INVALID_SPEC, "NULL output");
    MW_TRY({
        std::vector<int64_t> o(k > 0 ? k : 0), l(k > 0 ? k : 0);
        mw_status st = mw::partition_plan(L, g, fractions, k, strict != 0, o.data(), l.data());
        if (st) return st;
        for (int i = 0; i < k; ++i) {
            offsets[i] = o[i];
            lengths[i] = l[i];
        }
        return MW_OK;
    })
}

void mw_balance_defaults(mw_balance_params* p) {
    if (!p) return;
    p->weight = 2.0 / 3.0;
    p->max_dev = 0.85;
    p->c_factor = 1.0;
    p->trigger = 0.95;
    p->mode = MW_BALANCE_PROPORTIONAL;
}

mw_status mw_balance_step(const mw_balance_params* p, mw_balance_state* inout,
                          const float* per_part_ms, const int64_t* per_part_len,
                          const double* cur, int32_t n, double* next, int32_t* triggered) {
    if (!p || !inout || !triggered || !next) return fail(MW_E_INVALID_SPEC, "NULL argument");
    MW_TRY({
        mw_balance_state s = *inout;
        std::vector<double> nx(n > 0 ? n : 0);
        int trig = 0;
        mw_status st = mw::balance_step(*p, s, per_part_ms, per_part_len, cur, n, nx.data(), &trig);
        if (st) return st;
        *inout = s;
        for (int i = 0; i < n; ++i) next[i] = nx[i];
        *triggered = trig;
        return MW_OK;
    })
}

const char* mw_status_string(mw_status s) {
    switch (s) {
        case MW_OK: return "MW_OK";
        case MW_E_INVALID_SPEC: return "MW_E_INVALID_SPEC";
        case MW_E_EPU_NU: return "MW_E_EPU_NU";
        case MW_E_INFEASIBLE_PARTITION: return "MW_E_INFEASIBLE_PARTITION";
        case MW_E_SHAPE_MISMATCH: return "MW_E_SHAPE_MISMATCH";
        case MW_E_MISSING_ITERATION_COUNT: return "MW_E_MISSING_ITERATION_COUNT";
        case MW_E_NOT_CONVERGED: return "MW_E_NOT_CONVERGED";
        case MW_E_CUDA: return "MW_E_CUDA";
        case MW_E_NCCL: return "MW_E_NCCL";
        case MW_E_STATE: return "MW_E_STATE";
        case MW_E_OOM: return "MW_E_OOM";
        case MW_E_UNSUPPORTED: return "MW_E_UNSUPPORTED";
    }
    return "MW_E_UNKNOWN";
}

int32_t mw_abi_version(void) { return MW_ABI_VERSION; }

}  // extern "C"
