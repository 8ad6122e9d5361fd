// sct.h — host-side skeleton computation tree IR, fusion planner,
// partitioner and balancer of libmarrow (internal; the ABI is marrow.h).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "marrow.h"

namespace mw {

// ------------------------------------------------------------ errors
struct Error {
    mw_status code;
    std::string msg;
};
void set_error(const std::string& msg);
mw_status fail(mw_status code, const std::string& msg);

// ------------------------------------------------------------ tree
enum class NodeType { Leaf, Pipeline, Map, MapReduce, LoopFor, LoopWhile, LoopHost };
enum class LeafKind {
    Saxpy, GaussNoise, Solarize, Mirror, Segment, HystStep, HystFinalize,
    NbodyStep, NbodyAccel, MapIdentity, MapProduct, DebugTraits, Fft, Reduce,
    TermMap,     // reduction-stage term map (ia: MW_TERM_*)
    ScalarMap    // reduction-stage map of the reduced value (ia: MW_SCALAR_*, ib: bits of c)
};

struct Step;
struct NodeCache;   // per-node run plan, computed once (see plan_cached)

struct Node {
    int refs = 1;
    std::atomic<NodeCache*> cache{nullptr};   // immutable once published
    NodeType type = NodeType::Leaf;
    // leaf
    LeafKind leaf = LeafKind::Saxpy;
    float fa = 0.f, fb = 0.f;          // saxpy a | nbody dt, eps2
    int64_t ia = 0, ib = 0, ic = 0;    // seed/scale | T | lo/hi | epu/nu/strict
    // composites
    std::vector<Node*> kids;
    int64_t n = 0;                     // LoopFor count | LoopWhile max_iters
    int32_t check_every = 1;
    int32_t merge_op = 0;
    void* fn = nullptr;                // MapReduce USER merge | LoopHost condition
    void* user = nullptr;
    int32_t in_kind = 0, out_kind = 0; // MW_VK_*
};

void retain(Node* n);
void release(Node* n);
std::string canonical(const Node* n);
void leaf_epu_nu(const Node* leaf, int64_t* epu, int64_t* nu);
std::vector<const Node*> leaves(const Node* n);

// ------------------------------------------------------------ fusion plan
// The tree flattened into the sequence of executable steps; adjacent
// element-/row-local stages of the same value kind are merged into ONE
// fused chain (they share the partitioning, so their
// intermediates never leave the device — here, never leave registers).
enum class StepKind { Saxpy, Rgba, U8, StencilFor, StencilWhile, NbodyLoop, NbodyAccel,
                      MapStage, Reduce, Traits, Fft };
struct ChainOp {
    LeafKind kind;
    float fa;
    int64_t ia, ib;
};
struct Step {
    StepKind kind;
    std::vector<ChainOp> ops;
    int64_t n = 0;                     // StencilWhile: max STEPS (= max body executions x m)
    int64_t m = 1;                     // StencilWhile: steps per body execution
    int32_t check_every = 1;
    float dt = 0.f, eps2 = 0.f;
    bool dot = false;
    int64_t epu = 1, nu = 1;
    bool strict = false;
    int32_t merge_op = 0;              // Reduce: MW_MERGE_*
    int32_t reduce_op = 0;             // Reduce: MW_REDUCE_* (device reduction stage)
    std::vector<ChainOp> pre;          // Reduce: saxpy chain fused into the map stage (dot)
    int32_t term_map = -1;             // Reduce: -1 none, else MW_TERM_* applied to every term
    std::vector<std::pair<int32_t, double>> post;   // Reduce: MW_SCALAR_* maps of the result
    void* fn = nullptr;
    void* user = nullptr;
};
mw_status plan(const Node* root, std::vector<Step>* out);

// The plan, granule and strict flag of a node depend only on the (immutable)
// tree: computed on first use and published once (compare-exchange), so
// repeated runs of a tree skip the planner.  Returns nullptr + *st on error.
struct NodeCache {
    std::vector<Step> prog;
    int64_t granule = 1;
    bool strict = false;
    mw_status gst = MW_OK;   // granule status (reported when the plan is run)
};
const NodeCache* plan_cached(const Node* root, mw_status* st);

// ------------------------------------------------------------ partitioner / balancer
int64_t granule_of(const Node* root, mw_status* st);
bool strict_of(const Node* root);
mw_status partition_plan(int64_t L, int64_t g, const double* d, int k, bool strict,
                         int64_t* off, int64_t* len);
mw_status check_distribution(const double* d, int k);
mw_status balance_step(const mw_balance_params& p, mw_balance_state& s, const float* ms,
                       const int64_t* len, const double* cur, int n, double* next, int* trig);

void sha256(const void* data, size_t len, uint8_t out[32]);

}  // namespace mw
