// Host planner: symbolic H-Cholesky / forward-solve / sampler (PAPER.md
// sec. 3.1-3.2, l.259-283) lowered to a DAG of device tasks, levelled into
// waves.  The plan depends only on the geometry (tree, partition, leaf, eta,
// kmax) -- never on theta -- so it is built once per location set and replayed
// for every likelihood evaluation; ranks are read by the kernels at run time
// from rank slots in device memory.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "hm_tasks.h"
#include "tree.h"

namespace hm {

// storage of one lower block of the partition
enum StoreKind : int32_t { ST_SUB = 0, ST_DENSE = 1, ST_LR = 2 };

struct BStore {
    int32_t kind = ST_SUB;
    int32_t m = 0, p = 0;        // rows |t|, cols |s|
    int64_t d_off = -1;          // dense m x p (ld m)
    int64_t u_off = -1, v_off = -1;
    int32_t cap = 0, rslot = -1;
    int32_t d_res = -1;          // resource id (dense)
    int32_t u_res0 = -1, v_res0 = -1;  // first leaf-chunk resource of U (rows t) / V (rows s)
    int64_t inv_off = -1;        // diagonal leaf blocks: L^{-1} (m x m) written with the factor
    int32_t inv_res = -1;
    int64_t x_off = -1;          // dense leaf block (c1, c0) of a two-leaf diagonal cluster c:
    int32_t x_res = -1;          // X10 = -L11^{-1} L10 L00^{-1} (|c1| x |c0|), the off-diagonal
                                 // block of L_cc^{-1}, so a forward solve over c is one task
};

// A matrix whose rows are the points of a cluster (tree order), split into
// row chunks at that cluster's leaf clusters for dependency tracking.
struct Thin {
    int64_t off = -1;
    int32_t ld = 0;
    int32_t cluster = -1;
    int32_t cols = 0;            // static (maximum) number of columns
    int32_t slot = -1;           // rank slot giving the actual column count (-1: static)
    int32_t res0 = -1;           // resource id of the chunk of the first leaf of `cluster`
    int32_t tmp = -1;            // temporary-arena allocation it lives in (-1: permanent storage)
};

struct Phase {                   // one executable phase (levelled task lists)
    std::vector<VIns> ins;
    std::vector<VTerm> terms;    // VM_MGEMM terms
    std::vector<VTask> vt;       // sorted by wave
    std::vector<TTask> tt;       // sorted by wave
    std::vector<TPiece> tp;
    std::vector<int32_t> v_wave_begin, t_wave_begin;  // size nwaves + 1
    std::vector<XTask> xt;       // every task, topological (wave) order
    std::vector<int32_t> xdeps;  // predecessor positions in xt
    int32_t n_bars = 0;          // group barriers of cooperative truncations
    int32_t nwaves = 0;
    int64_t n_launches() const;
};

struct Plan {
    // geometry-derived layout
    std::vector<BStore> bs;
    std::vector<int32_t> diag_of;      // cluster -> diagonal block id
    std::vector<int32_t> leaf_begin;   // cluster -> index of its first leaf cluster
    std::vector<int32_t> leaf_count;
    std::vector<int32_t> leaf_cluster; // leaf index -> cluster id
    std::vector<int32_t> leaf_diag_idx;// leaf index -> logd index (== leaf index)
    int32_t n_leaves = 0;
    int32_t n_slots = 0;
    int32_t kmax = 0;
    int64_t pool_blocks = 0;           // doubles used by block storage (C~ / L~)
    int64_t pool_total = 0;            // doubles incl. temporaries and workspaces
    int64_t logd_off = 0;              // n_leaves doubles
    int64_t z_off = 0;                 // solve RHS buffer: n x ZW (col-major, ld n)
    int32_t zw = 64;
    int32_t z_slot = -1;               // rank slot holding the active column count of the z buffer
                                       // (set by hm_loglik / hm_sample before the phase runs)
    int64_t bytes_C = 0;               // bytes of block storage at capacity
    int64_t ring_off = 0, ring_size = 0;  // truncation workspace ring (doubles)
    int64_t tmp_off = 0;                  // ring of 64 x 64 temporary tiles (split dense updates)
    int64_t arena_off = 0, arena_size = 0;   // temporaries of the H x thin products (liveness-planned)
    // assembly
    std::vector<DenseGenTask> dgen;
    std::vector<AcaTask> aca;
    Phase recompress;                  // TRUNC of every LR block after ACA
    // factorisation and solves
    Phase chol;
    Phase solve;                       // v <- L~^{-1} z  on the z buffer
    Phase lmul;                        // z <- L~ z       (sampler)
    int64_t n_tasks_chol = 0;
    int64_t n_split = 0;               // Cholesky truncations split into partial merge + final step
    int32_t n_block_slots = 0;         // rank slots [0, n_block_slots) belong to blocks (+ z_slot)
    std::string summary() const;
};

// Largest dense leaf block the tile VM handles in one 64 x 64 tile; trees with larger
// leaves or leaves at several depths are planned on refine_for_plan's storage tree.
constexpr int32_t TILE_MAX_LEAF = 64;

// Build the full plan for a tree (any n >= 1, any leaf size the storage refinement can
// halve down to TILE_MAX_LEAF without empty clusters).
// arena_budget: doubles the H x thin temporaries may occupy before recycling memory
// whose last users finish late (longer critical path, smaller footprint).
// cap_hint (optional, indexed like Plan::bs): per-block rank capacity below kmax (adaptive
// capacities, hm_params.adaptive_cap).  assembly_only: plan only the assembly and the
// recompression (a rank probe), no Cholesky / solve / sampler phases.
void build_plan(const Tree& T, int32_t kmax, Plan& P, int32_t coop_max = TR_COOP_DEFAULT,
                int64_t arena_budget = INT64_MAX, const std::vector<int32_t>* cap_hint = nullptr,
                bool assembly_only = false);

}  // namespace hm
