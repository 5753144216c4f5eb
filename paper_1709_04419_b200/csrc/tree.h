// Host-side geometry: cluster tree T_I and block cluster tree T_{IxI}
// (sec. 2.1, Definition 1, l.152-160; leaf size n_min l.211).
// Readings R1-R3 of DESIGN.md sec. 3.  Compiled with -ffp-contract=off so the
// admissibility decisions are bit-identical to any other IEEE evaluation of
// the same expressions.
#pragma once
#include <cstdint>
#include <vector>

namespace hm {

struct Cluster {
    int64_t lo, hi;       // [lo, hi) in tree order
    int32_t level;
    int32_t parent;
    int32_t child[2];     // -1 if leaf
    double bmin[2], bmax[2];
    int64_t size() const { return hi - lo; }
    bool leaf() const { return child[0] < 0; }
};

enum BlockKind : int32_t { BK_SUB = 0, BK_DENSE = 1, BK_LR = 2 };

// A block of the LOWER part of the block cluster tree (t >= s in tree order),
// including the diagonal blocks (t, t).
struct Block {
    int32_t t, s;         // cluster ids (row, column)
    int32_t kind;         // BlockKind in the partition of C~
    int32_t admissible;   // partition flag (1 = admissible leaf)
    int32_t level;
    int32_t parent;
    int32_t child[4];     // SUB off-diagonal: (t0,s0),(t1,s0),(t0,s1),(t1,s1);
                          // SUB diagonal:    (t0,t0),(t1,t0),(t1,t1), -1
};

struct Tree {
    int64_t n = 0;
    int32_t leaf = 0;
    double eta = 0;
    std::vector<Cluster> clusters;     // pre-order, root = 0
    std::vector<int64_t> perm;         // perm[k] = original index of k-th point
    std::vector<double> pts;           // tree-ordered points (2n)
    std::vector<Block> blocks;         // lower part, root block = 0
    std::vector<int64_t> full_blocks;  // full partition, 6 ints per leaf block (oracle order)
    int32_t depth = 0;
    int64_t n_leaf_clusters = 0;
};

// Throws std::invalid_argument on bad input.
void build_tree(const double* locs, int64_t n, int32_t leaf, double eta, Tree& T);

bool admissible(const Cluster& t, const Cluster& s, double eta);

// Storage tree for the planner.  The tile VM works on dense blocks of at most
// `maxleaf` rows and the Cholesky recursion pairs equal-depth leaves, while
// the paper's tree (Def. 1 with n_min, reading R1) may hold leaves at two
// depths (n / 2^l straddling n_min) and leaves above maxleaf (n_min up to 128,
// Table 1 l.213).  R refines every leaf of T by halving its index range
// (no reordering: tree order and perm are unchanged) until all leaves sit at
// one depth with at most maxleaf points, and splits every dense block of T's
// partition accordingly into dense sub-blocks.  Admissible (low-rank) blocks,
// their clusters and T's partition of I x I are untouched, so C~ is the same
// matrix; only the granularity of its dense part changes.  R.full_blocks is
// empty (the partition is T's).  Throws std::invalid_argument if a leaf would
// have to be split below one point.
void refine_for_plan(const Tree& T, int32_t maxleaf, Tree& R);
// true when T already has all leaves at one depth with at most maxleaf points
bool plan_ready(const Tree& T, int32_t maxleaf);

}  // namespace hm
