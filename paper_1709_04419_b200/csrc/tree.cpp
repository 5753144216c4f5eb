// Cluster tree + block cluster tree, sec. 2.1 (see tree.h).
#include "tree.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace hm {

static double diameter(const Cluster& c) {
    double dx = c.bmax[0] - c.bmin[0];
    double dy = c.bmax[1] - c.bmin[1];
    return std::sqrt(dx * dx + dy * dy);
}

static double distance(const Cluster& t, const Cluster& s) {
    double dx = std::max(0.0, std::max(s.bmin[0] - t.bmax[0], t.bmin[0] - s.bmax[0]));
    double dy = std::max(0.0, std::max(s.bmin[1] - t.bmax[1], t.bmin[1] - s.bmax[1]));
    return std::sqrt(dx * dx + dy * dy);
}

// Reading R2: admissible iff dist > 0 and min(diam t, diam s) <= eta * dist.
bool admissible(const Cluster& t, const Cluster& s, double eta) {
    double d = distance(t, s);
    return d > 0.0 && std::min(diameter(t), diameter(s)) <= eta * d;
}

namespace {

struct Builder {
    const double* P;   // original points, row-major n x 2
    int32_t leaf;
    std::vector<int64_t>& perm;
    std::vector<Cluster>& cl;
    int32_t depth = 0;

    int32_t rec(int64_t lo, int64_t hi, int32_t level, int32_t parent) {
        Cluster c;
        c.lo = lo; c.hi = hi; c.level = level; c.parent = parent;
        c.child[0] = c.child[1] = -1;
        double x0 = P[2 * perm[lo]], y0 = P[2 * perm[lo] + 1];
        c.bmin[0] = c.bmax[0] = x0;
        c.bmin[1] = c.bmax[1] = y0;
        for (int64_t k = lo + 1; k < hi; ++k) {
            double x = P[2 * perm[k]], y = P[2 * perm[k] + 1];
            c.bmin[0] = std::min(c.bmin[0], x); c.bmax[0] = std::max(c.bmax[0], x);
            c.bmin[1] = std::min(c.bmin[1], y); c.bmax[1] = std::max(c.bmax[1], y);
        }
        int32_t id = (int32_t)cl.size();
        cl.push_back(c);
        depth = std::max(depth, level);
        int64_t m = hi - lo;
        if (m > leaf) {
            // R1: longest axis (first on ties), order by (coordinate, original index)
            double e0 = c.bmax[0] - c.bmin[0], e1 = c.bmax[1] - c.bmin[1];
            int axis = (e0 >= e1) ? 0 : 1;
            const double* PP = P;
            std::sort(perm.begin() + lo, perm.begin() + hi, [PP, axis](int64_t a, int64_t b) {
                double ca = PP[2 * a + axis], cb = PP[2 * b + axis];
                if (ca < cb) return true;
                if (cb < ca) return false;
                return a < b;
            });
            int64_t mid = lo + m / 2;
            int32_t c0 = rec(lo, mid, level + 1, id);
            int32_t c1 = rec(mid, hi, level + 1, id);
            cl[id].child[0] = c0;
            cl[id].child[1] = c1;
        }
        return id;
    }
};

struct BlockBuilder {
    Tree& T;
    // Full partition in the oracle's recursion order (t-children outer loop).
    void full(int32_t t, int32_t s) {
        const Cluster& ct = T.clusters[t];
        const Cluster& cs = T.clusters[s];
        if (admissible(ct, cs, T.eta)) {
            push(ct, cs, 1);
        } else if (ct.leaf() || cs.leaf()) {
            push(ct, cs, 0);
        } else {
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) full(ct.child[i], cs.child[j]);
        }
    }
    void push(const Cluster& t, const Cluster& s, int adm) {
        int64_t v[6] = {t.lo, t.hi, s.lo, s.hi, t.level, adm};
        T.full_blocks.insert(T.full_blocks.end(), v, v + 6);
    }
    // Lower part (t >= s) as an explicit tree of Block records.
    int32_t lower(int32_t t, int32_t s, int32_t parent) {
        const Cluster& ct = T.clusters[t];
        const Cluster& cs = T.clusters[s];
        Block b;
        b.t = t; b.s = s; b.level = ct.level; b.parent = parent;
        for (int i = 0; i < 4; ++i) b.child[i] = -1;
        b.admissible = admissible(ct, cs, T.eta) ? 1 : 0;
        if (b.admissible) b.kind = BK_LR;
        else if (ct.leaf() || cs.leaf()) b.kind = BK_DENSE;
        else b.kind = BK_SUB;
        int32_t id = (int32_t)T.blocks.size();
        T.blocks.push_back(b);
        if (b.kind == BK_SUB) {
            const int32_t t0 = ct.child[0], t1 = ct.child[1];
            const int32_t s0 = cs.child[0], s1 = cs.child[1];
            if (t == s) {
                int32_t a = lower(t0, t0, id);
                int32_t c = lower(t1, t0, id);
                int32_t d = lower(t1, t1, id);
                T.blocks[id].child[0] = a; T.blocks[id].child[1] = c; T.blocks[id].child[2] = d;
            } else {
                int32_t a = lower(t0, s0, id);
                int32_t c = lower(t1, s0, id);
                int32_t d = lower(t0, s1, id);
                int32_t e = lower(t1, s1, id);
                T.blocks[id].child[0] = a; T.blocks[id].child[1] = c;
                T.blocks[id].child[2] = d; T.blocks[id].child[3] = e;
            }
        }
        return id;
    }
};

}  // namespace

void build_tree(const double* locs, int64_t n, int32_t leaf, double eta, Tree& T) {
    if (n < 1) throw std::invalid_argument("hm_tree_build: n >= 1 required");
    if (leaf < 1) throw std::invalid_argument("hm_tree_build: leaf >= 1 required");
    if (!(eta > 0.0)) throw std::invalid_argument("hm_tree_build: eta > 0 required");
    for (int64_t i = 0; i < 2 * n; ++i)
        if (!std::isfinite(locs[i])) throw std::invalid_argument("hm_tree_build: non-finite coordinate");
    T = Tree();
    T.n = n; T.leaf = leaf; T.eta = eta;
    T.perm.resize(n);
    for (int64_t i = 0; i < n; ++i) T.perm[i] = i;
    Builder B{locs, leaf, T.perm, T.clusters};
    B.rec(0, n, 0, -1);
    T.depth = B.depth;
    T.n_leaf_clusters = 0;
    for (auto& c : T.clusters) T.n_leaf_clusters += c.leaf() ? 1 : 0;
    T.pts.resize(2 * n);
    for (int64_t k = 0; k < n; ++k) {
        T.pts[2 * k] = locs[2 * T.perm[k]];
        T.pts[2 * k + 1] = locs[2 * T.perm[k] + 1];
    }
    BlockBuilder BB{T};
    BB.full(0, 0);
    BB.lower(0, 0, -1);
}

bool plan_ready(const Tree& T, int32_t maxleaf) {
    int32_t d = -1;
    for (const Cluster& c : T.clusters) {
        if (!c.leaf()) continue;
        if (c.size() > maxleaf) return false;
        if (d < 0) d = c.level;
        else if (d != c.level) return false;
    }
    return true;
}

namespace {

struct Refiner {
    const Tree& T;
    Tree& R;
    int32_t D = 0;                     // common leaf depth of R
    std::vector<int32_t> map;          // T cluster -> R cluster

    void bbox(Cluster& c) const {
        c.bmin[0] = c.bmax[0] = T.pts[2 * c.lo];
        c.bmin[1] = c.bmax[1] = T.pts[2 * c.lo + 1];
        for (int64_t k = c.lo + 1; k < c.hi; ++k) {
            c.bmin[0] = std::min(c.bmin[0], T.pts[2 * k]); c.bmax[0] = std::max(c.bmax[0], T.pts[2 * k]);
            c.bmin[1] = std::min(c.bmin[1], T.pts[2 * k + 1]); c.bmax[1] = std::max(c.bmax[1], T.pts[2 * k + 1]);
        }
    }
    // virtual subtree below a refined leaf: index halving down to depth D
    int32_t virt(int64_t lo, int64_t hi, int32_t level, int32_t parent) {
        if (hi <= lo) throw std::invalid_argument("refine_for_plan: a leaf would be split below one point");
        Cluster c;
        c.lo = lo; c.hi = hi; c.level = level; c.parent = parent;
        c.child[0] = c.child[1] = -1;
        bbox(c);
        const int32_t id = (int32_t)R.clusters.size();
        R.clusters.push_back(c);
        if (level < D) {
            const int64_t mid = lo + (hi - lo) / 2;
            const int32_t a = virt(lo, mid, level + 1, id);
            const int32_t b = virt(mid, hi, level + 1, id);
            R.clusters[id].child[0] = a;
            R.clusters[id].child[1] = b;
        }
        return id;
    }
    int32_t copy(int32_t t, int32_t parent) {
        const Cluster& ct = T.clusters[t];
        Cluster c = ct;
        c.parent = parent;
        const int32_t id = (int32_t)R.clusters.size();
        map[t] = id;
        if (ct.leaf() && ct.level < D) return virt(ct.lo, ct.hi, ct.level, parent);   // == id
        R.clusters.push_back(c);
        if (ct.leaf()) return id;
        const int32_t a = copy(ct.child[0], id);
        const int32_t b = copy(ct.child[1], id);
        R.clusters[id].child[0] = a;
        R.clusters[id].child[1] = b;
        return id;
    }
    // R block for the cluster pair (t, s) of R; tb = T block it stands for (or -1 inside a
    // split dense block, which is dense all the way down)
    int32_t block(int32_t tb, int32_t t, int32_t s, int32_t parent) {
        const Cluster& ct = R.clusters[t];
        const Cluster& cs = R.clusters[s];
        Block b;
        b.t = t; b.s = s; b.level = ct.level; b.parent = parent;
        for (int i = 0; i < 4; ++i) b.child[i] = -1;
        if (tb >= 0) {
            const Block& o = T.blocks[tb];
            b.admissible = o.admissible;
            b.kind = o.kind;
        } else {
            b.admissible = 0;
            b.kind = BK_DENSE;
        }
        if (b.kind == BK_DENSE && !(ct.leaf() && cs.leaf())) b.kind = BK_SUB;   // split dense block
        const int32_t id = (int32_t)R.blocks.size();
        R.blocks.push_back(b);
        if (b.kind != BK_SUB) return id;
        const bool orig_sub = tb >= 0 && T.blocks[tb].kind == BK_SUB;
        auto ch = [&](int k) { return orig_sub ? T.blocks[tb].child[k] : -1; };
        const int32_t t0 = ct.child[0], t1 = ct.child[1], s0 = cs.child[0], s1 = cs.child[1];
        if (t == s) {
            const int32_t a = block(ch(0), t0, t0, id);
            const int32_t c = block(ch(1), t1, t0, id);
            const int32_t d = block(ch(2), t1, t1, id);
            R.blocks[id].child[0] = a; R.blocks[id].child[1] = c; R.blocks[id].child[2] = d;
        } else {
            const int32_t a = block(ch(0), t0, s0, id);
            const int32_t c = block(ch(1), t1, s0, id);
            const int32_t d = block(ch(2), t0, s1, id);
            const int32_t e = block(ch(3), t1, s1, id);
            R.blocks[id].child[0] = a; R.blocks[id].child[1] = c;
            R.blocks[id].child[2] = d; R.blocks[id].child[3] = e;
        }
        return id;
    }
};

}  // namespace

void refine_for_plan(const Tree& T, int32_t maxleaf, Tree& R) {
    if (maxleaf < 1) throw std::invalid_argument("refine_for_plan: maxleaf >= 1 required");
    Refiner F{T, R};
    // common depth: every leaf needs ceil(log2(size / maxleaf)) halvings
    for (const Cluster& c : T.clusters) {
        if (!c.leaf()) continue;
        int32_t k = 0;
        int64_t s = c.size();
        while (s > maxleaf) {
            s = (s + 1) / 2;
            ++k;
        }
        F.D = std::max(F.D, c.level + k);
    }
    R = Tree();
    R.n = T.n; R.leaf = T.leaf; R.eta = T.eta;
    R.perm = T.perm;
    R.pts = T.pts;
    F.map.assign(T.clusters.size(), -1);
    F.copy(0, -1);
    R.depth = F.D;
    R.n_leaf_clusters = 0;
    for (auto& c : R.clusters) R.n_leaf_clusters += c.leaf() ? 1 : 0;
    // T's block records refer to T's cluster ids: walk both trees together (R's root is 0,
    // and the children of every non-leaf T cluster keep their order in R)
    F.block(0, 0, 0, -1);
    for (const Block& b : R.blocks)
        if (b.kind == BK_SUB && b.child[0] < 0) throw std::logic_error("refine_for_plan: SUB block without children");
}

}  // namespace hm
