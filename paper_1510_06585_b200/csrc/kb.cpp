// kb.cpp — Knowledge Base and profile building (NEXT-2), host side.
//
// The paper's decision process (Fig. 5) keeps, per SCT and
// workload, the best configuration found so far (profile items (a)-(f),
// P:446-456) and derives configurations for unseen workloads by narrowing
// the scope SCT -> workload -> dimensionality.  Profile building
// (Alg. 1) searches the configuration space by running the SCT.
// On B200 the searched "platform configuration" is the set of kernel tuning
// knobs (MW_TUNE_*) plus the distribution vector; every knob value gives
// bit-identical results, so the search only changes speed.
//
// Reading R22: the paper interpolates with Alglib Fast RBF for
// 1-3 dimensions and Euclidean nearest neighbour above; the knobs here are
// discrete, so derivation is nearest neighbour in log2-size space at every
// dimensionality (an RBF would interpolate between categorical settings).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "marrow.h"
#include "mw_kernels.h"
#include "sct.h"

using mw::fail;

namespace {

struct Record {
    std::string sct;               // hex SHA-256 of the tree (item a)
    std::vector<int64_t> dims;     // workload characterization (item b)
    std::vector<double> dist;      // per-partition fractions (item c)
    int tune[MW_TUNE_COUNT];       // platform configuration (item d)
    double ms;                     // best time (item e)
    int prov;                      // provenance (item f)
};

std::string hex_id(const mw_node* root) {
    uint8_t id[32];
    mw_node_id(root, id);
    static const char* H = "0123456789abcdef";
    std::string s;
    for (int i = 0; i < 32; ++i) {
        s += H[id[i] >> 4];
        s += H[id[i] & 15];
    }
    return s;
}

double dist_log2(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
    double d = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double x = std::log2((double)std::max<int64_t>(1, a[i]));
        const double y = std::log2((double)std::max<int64_t>(1, b[i]));
        d += (x - y) * (x - y);
    }
    return std::sqrt(d);
}

}  // namespace

struct mw_kb {
    std::string path;
    std::vector<Record> recs;
};

extern "C" {

mw_status mw_kb_open(const char* path, mw_kb** out) {
    if (!out) return fail(MW_E_INVALID_SPEC, "out is NULL");
    try {
        mw_kb* kb = new mw_kb;
        kb->path = path ? path : "";
        if (path && *path) {
            std::ifstream f(path);
            std::string line;
            while (std::getline(f, line)) {
                if (line.empty() || line[0] == '#') continue;
                std::istringstream is(line);
                Record r;
                int nd = 0, np = 0;
                if (!(is >> r.sct >> nd) || nd < 0 || nd > 8) continue;
                r.dims.resize(nd);
                for (auto& d : r.dims) is >> d;
                is >> np;
                if (np < 0 || np > 4096) continue;
                r.dist.resize(np);
                for (auto& x : r.dist) is >> x;
                int nt = 0;
                is >> r.prov >> r.ms >> nt;
                if (nt < 0 || nt > 64) continue;
                mwk::tune_defaults(r.tune);   // knobs added after the record was written
                for (int k = 0; k < nt; ++k) {
                    int v = 0;
                    is >> v;
                    if (k < MW_TUNE_COUNT) r.tune[k] = v;
                }
                if (is) kb->recs.push_back(r);
            }
        }
        *out = kb;
        return MW_OK;
    } catch (...) {
        return fail(MW_E_OOM, "knowledge base allocation failed");
    }
}

mw_status mw_kb_save(const mw_kb* kb) {
    if (!kb) return fail(MW_E_STATE, "NULL kb");
    if (kb->path.empty()) return MW_OK;
    std::ofstream f(kb->path, std::ios::trunc);
    if (!f) return fail(MW_E_INVALID_SPEC, "cannot write knowledge base file " + kb->path);
    f << "# marrow knowledge base v1: sct_id ndims dims.. nparts fractions.. provenance best_ms "
         "ntune tune..\n";
    char buf[64];
    for (const Record& r : kb->recs) {
        f << r.sct << ' ' << r.dims.size();
        for (auto d : r.dims) f << ' ' << d;
        f << ' ' << r.dist.size();
        for (auto x : r.dist) {
            snprintf(buf, sizeof buf, " %.17g", x);
            f << buf;
        }
        snprintf(buf, sizeof buf, " %d %.9g %d", r.prov, r.ms, (int)MW_TUNE_COUNT);
        f << buf;
        for (int k = 0; k < MW_TUNE_COUNT; ++k) f << ' ' << r.tune[k];
        f << '\n';
    }
    return f ? MW_OK : fail(MW_E_INVALID_SPEC, "write failed: " + kb->path);
}

mw_status mw_kb_close(mw_kb* kb) {
    if (!kb) return fail(MW_E_STATE, "NULL kb");
    mw_status st = mw_kb_save(kb);
    delete kb;
    return st;
}

mw_status mw_kb_count(const mw_kb* kb, int32_t* n) {
    if (!kb || !n) return fail(MW_E_INVALID_SPEC, "NULL argument");
    *n = (int32_t)kb->recs.size();
    return MW_OK;
}

mw_status mw_kb_store(mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                      const int32_t* tune, const double* fractions, int32_t nparts,
                      double best_ms, int32_t provenance) {
    if (!kb || !root || (ndims > 0 && !dims) || !tune || (nparts > 0 && !fractions))
        return fail(MW_E_INVALID_SPEC, "NULL argument");
    if (ndims < 0 || ndims > 8 || nparts < 0) return fail(MW_E_INVALID_SPEC, "bad sizes");
    Record r;
    r.sct = hex_id(root);
    r.dims.assign(dims, dims + ndims);
    r.dist.assign(fractions, fractions + nparts);
    for (int k = 0; k < MW_TUNE_COUNT; ++k) r.tune[k] = tune[k];
    r.ms = best_ms;
    r.prov = provenance;
    // progressive refinement: keep the best per (SCT, workload)
    for (Record& q : kb->recs)
        if (q.sct == r.sct && q.dims == r.dims) {
            if (best_ms < q.ms || q.prov == MW_PROV_DERIVED) q = r;
            return MW_OK;
        }
    kb->recs.push_back(r);
    return MW_OK;
}

mw_status mw_kb_find(const mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                     int32_t* found, int32_t* provenance, double* best_ms) {
    if (!kb || !root || (ndims > 0 && !dims) || !found) return fail(MW_E_INVALID_SPEC, "NULL argument");
    const std::string id = hex_id(root);
    const std::vector<int64_t> w(dims, dims + ndims);
    *found = 0;
    for (const Record& r : kb->recs)
        if (r.sct == id && r.dims == w) {
            *found = 1;
            if (provenance) *provenance = r.prov;
            if (best_ms) *best_ms = r.ms;
            break;
        }
    return MW_OK;
}

mw_status mw_kb_lookup(const mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                       int32_t* tune_out, double* fractions_out, int32_t nparts, int32_t* scope) {
    if (!kb || !root || (ndims > 0 && !dims) || !tune_out || !scope)
        return fail(MW_E_INVALID_SPEC, "NULL argument");
    const std::string id = hex_id(root);
    const std::vector<int64_t> w(dims, dims + ndims);
    const Record* best = nullptr;
    int sc = MW_KB_NONE;
    // scope narrowing: this SCT, then this workload, then this dimensionality
    for (int pass = 0; pass < 4 && !best; ++pass) {
        double bd = 1e300;
        for (const Record& r : kb->recs) {
            bool in = false;
            switch (pass) {
                case 0: in = r.sct == id && r.dims == w; break;
                case 1: in = r.sct == id && r.dims.size() == w.size(); break;
                case 2: in = r.dims == w; break;
                case 3: in = r.dims.size() == w.size(); break;
            }
            if (!in) continue;
            const double d = dist_log2(r.dims, w);
            if (d < bd) {
                bd = d;
                best = &r;
            }
        }
        if (best) sc = pass == 0 ? MW_KB_EXACT : (pass == 1 ? MW_KB_SCT : (pass == 2 ? MW_KB_WORKLOAD : MW_KB_DIMENSIONALITY));
    }
    *scope = sc;
    if (!best) return MW_OK;
    for (int k = 0; k < MW_TUNE_COUNT; ++k) tune_out[k] = best->tune[k];
    if (fractions_out && nparts > 0) {
        if ((int32_t)best->dist.size() == nparts)
            for (int i = 0; i < nparts; ++i) fractions_out[i] = best->dist[i];
        else
            for (int i = 0; i < nparts; ++i) fractions_out[i] = 1.0 / nparts;
    }
    return MW_OK;
}

}  // extern "C"
