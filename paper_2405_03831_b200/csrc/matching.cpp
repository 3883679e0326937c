// matching.cpp -- exact O(n^3) Edmonds blossom matching on a dense graph (host C++).
//
// Replaces matcher._max_weight_matching (matcher.py:180-542) behind
// matcher.min_weight_perfect_matching (matcher.py:78-88); see
// include/cosched_match.h.  Primal-dual method (Edmonds; Galil's survey):
// alternating trees grow from free vertices with S/T labels, tight S-S edges
// close blossoms or augment, and when the search stalls the duals move by
// the smallest of the four deltas.  Vertex duals are stored doubled so the
// S-S delta (slack / 2) stays integral; all arithmetic is on 128-bit integers
// obtained by scaling the double weights by a power of two, so "tight" means
// slack == 0 exactly.  The solver runs on an adjacency (CSR) graph whose
// edges carry their scaled integer weights.
//
// Minimum-weight perfect matching of the complete graph (cm_min_weight_perfect_
// matching*) is solved as a maximum-weight PERFECT matching (certified_perfect):
// an eps-scaling auction on the assignment relaxation prices the vertices
// (row-parallel, a persistent host thread pool), the prices give exact integer
// duals feasible on every edge, the blossom solver runs warm from those duals
// on a SPARSE candidate graph -- the k least-slack edges of every vertex -- and
// its LP dual is then certified on the complete graph: every edge's reduced
// cost y_i + y_j + sum of the duals of the blossoms containing both ends - w_ij
// must be >= 0 (the reference's verify-optimum condition).  Violating edges
// are added and the solve resumes from the previous duals and matching, so the
// result is a certified optimum of the full graph (~2 s at n = 4,096 instead
// of hours).  The dense O(n^2) scans run in double and re-check near-ties in
// i128, so every feasibility and tightness fact is exact.
#include "cosched_match.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

namespace {

typedef __int128 i128;

struct Edge {          // oriented edge: a -> b (vertices); a < 0 means "none"
    int32_t a = -1, b = -1;
    i128 w = 0;        // scaled integer weight (best-edge candidates only)
    bool none() const { return a < 0; }
};

// undirected graph in CSR form, both directions stored
struct Graph {
    int n = 0;
    std::vector<int64_t> off;
    std::vector<int32_t> nbr;
    std::vector<i128> w;
};

class Blossom {
public:
    explicit Blossom(const Graph &g) : n_(g.n), g_(g) {
        const int n = g.n;
        const int N2 = 2 * n;
        mate_.assign(n, -1);
        label_.assign(N2, 0);
        labeledge_.assign(N2, Edge());
        inblossom_.resize(n);
        for (int v = 0; v < n; ++v) inblossom_[v] = v;
        parent_.assign(N2, -1);
        childs_.assign(N2, {});
        edges_.assign(N2, {});
        base_.assign(N2, -1);
        for (int v = 0; v < n; ++v) base_[v] = v;
        bestedge_.assign(N2, Edge());
        bestlist_.assign(N2, {});
        has_bestlist_.assign(N2, 0);
        for (int b = N2 - 1; b >= n; --b) unused_.push_back(b);
        dual_.assign(N2, 0);
        allow_.assign((size_t)n * n, 0);
    }

    // Warm start (perfect-matching mode only): vertex duals in the solver's
    // doubled units at scale `extra`, and a matching whose edges are tight
    // under them; no blossoms.  Every edge of the graph must have slack >= 0.
    void warm(const std::vector<i128> &dual, const std::vector<int> &mate, int extra) {
        extra_ = extra;
        for (int v = 0; v < n_; ++v) { dual_[v] = dual[v]; mate_[v] = mate[v]; }
        warm_ = true;
    }

    int run(bool max_cardinality) {
        const int n = n_;
        if (!warm_) {
            // initial duals: doubled vertex duals = max weight (the reference init)
            i128 maxw = 0;
            for (const i128 &x : g_.w) maxw = std::max(maxw, x << extra_);
            for (int v = 0; v < n; ++v) dual_[v] = maxw;
        }

        for (int stage = 0; stage < n; ++stage) {
            std::fill(label_.begin(), label_.end(), 0);
            std::fill(bestedge_.begin(), bestedge_.end(), Edge());
            for (int b = n; b < 2 * n; ++b) { bestlist_[b].clear(); has_bestlist_[b] = 0; }
            clear_allow();
            queue_.clear();
            for (int v = 0; v < n; ++v)
                if (mate_[v] < 0 && label_[inblossom_[v]] == 0) assign_label(v, 1, -1);
            bool augmented = false;
            for (;;) {
                while (!queue_.empty() && !augmented) {
                    const int v = queue_.back();
                    queue_.pop_back();
                    augmented = scan_vertex(v);
                }
                if (augmented) break;
                // ---- choose delta ----
                int dtype = -1;
                i128 delta = 0;
                Edge dedge;
                int dblossom = -1;
                if (!max_cardinality) {
                    dtype = 1;
                    delta = dual_[0];
                    for (int v = 1; v < n; ++v) delta = std::min(delta, dual_[v]);
                }
                for (int v = 0; v < n; ++v) {
                    if (label_[inblossom_[v]] == 0 && !bestedge_[v].none()) {
                        i128 d = slack(bestedge_[v]);
                        if (dtype == -1 || d < delta) { delta = d; dtype = 2; dedge = bestedge_[v]; }
                    }
                }
                for (int b = 0; b < 2 * n; ++b) {
                    if (parent_[b] == -1 && base_[b] >= 0 && label_[b] == 1 && !bestedge_[b].none()) {
                        i128 ks = slack(bestedge_[b]);
                        if (ks & 1) { rescale(); ks = slack(bestedge_[b]); delta *= 2; }
                        i128 d = ks / 2;
                        if (dtype == -1 || d < delta) { delta = d; dtype = 3; dedge = bestedge_[b]; }
                    }
                }
                for (int b = n; b < 2 * n; ++b) {
                    if (base_[b] >= 0 && parent_[b] == -1 && label_[b] == 2 &&
                        (dtype == -1 || dual_[b] < delta)) {
                        delta = dual_[b]; dtype = 4; dblossom = b;
                    }
                }
                if (dtype == -1) {   // max-cardinality only: no further progress possible
                    dtype = 1;
                    delta = dual_[0];
                    for (int v = 1; v < n; ++v) delta = std::min(delta, dual_[v]);
                    if (delta < 0) delta = 0;
                }
                // ---- update duals ----
                for (int v = 0; v < n; ++v) {
                    int l = label_[inblossom_[v]];
                    if (l == 1) dual_[v] -= delta;
                    else if (l == 2) dual_[v] += delta;
                }
                for (int b = n; b < 2 * n; ++b) {
                    if (base_[b] >= 0 && parent_[b] == -1) {
                        if (label_[b] == 1) dual_[b] += delta;
                        else if (label_[b] == 2) dual_[b] -= delta;
                    }
                }
                if (dtype == 1) break;
                if (dtype == 2) {
                    set_allow(dedge.a, dedge.b);
                    int i = dedge.a, j = dedge.b;
                    if (label_[inblossom_[i]] == 0) std::swap(i, j);
                    queue_.push_back(i);
                } else if (dtype == 3) {
                    set_allow(dedge.a, dedge.b);
                    queue_.push_back(dedge.a);
                } else {
                    expand(dblossom, false);
                }
            }
            if (!augmented) break;
            for (int b = n; b < 2 * n; ++b)
                if (parent_[b] == -1 && base_[b] >= 0 && label_[b] == 1 && dual_[b] == 0)
                    expand(b, true);
        }
        return 0;
    }

    const std::vector<int> &mate() const { return mate_; }
    const std::vector<i128> &duals() const { return dual_; }
    const std::vector<int> &parents() const { return parent_; }
    int extra() const { return extra_; }

private:
    // ---- weights ----------------------------------------------------------
    i128 slack_w(int u, int v, i128 w) const { return dual_[u] + dual_[v] - 2 * (w << extra_); }
    i128 slack(const Edge &e) const { return slack_w(e.a, e.b, e.w); }
    bool allowed(int u, int v) const { return allow_[idx(u, v)]; }
    void set_allow(int u, int v) {
        const size_t k = idx(u, v);
        if (!allow_[k]) { allow_[k] = 1; touched_.push_back(k); }
    }
    void clear_allow() {
        for (size_t k : touched_) allow_[k] = 0;
        touched_.clear();
    }
    size_t idx(int u, int v) const { return u < v ? (size_t)u * n_ + v : (size_t)v * n_ + u; }

    // doubling every weight and dual keeps every relation; used if an S-S
    // slack is ever odd (so slack / 2 would not be exact)
    void rescale() {
        ++extra_;
        for (auto &d : dual_) d *= 2;
    }

    template <class F>
    void leaves(int b, F &&f) const {
        if (b < n_) { f(b); return; }
        for (int c : childs_[b]) leaves(c, f);
    }

    // ---- labels -----------------------------------------------------------
    // assign label t (1 = S, 2 = T) to the top blossom of w, reached from vertex p
    void assign_label(int w, int t, int p) {
        const int b = inblossom_[w];
        label_[w] = label_[b] = t;
        Edge e;                                  // (remote p, inside w); none for roots
        if (p >= 0) { e.a = p; e.b = w; }
        labeledge_[w] = labeledge_[b] = e;
        bestedge_[w] = bestedge_[b] = Edge();
        if (t == 1) {
            leaves(b, [this](int v) { queue_.push_back(v); });
        } else {
            const int bs = base_[b];
            assign_label(mate_[bs], 1, bs);
        }
    }

    // walk up from v and w; return the base of the new blossom or -1 (augmenting path)
    int scan_blossom(int v, int w) {
        std::vector<int> path;
        int found = -1;
        while (v != -1 || w != -1) {
            if (v != -1) {
                int b = inblossom_[v];
                if (label_[b] & 4) { found = base_[b]; break; }
                path.push_back(b);
                label_[b] = 5;
                if (labeledge_[b].none()) {
                    v = -1;
                } else {
                    v = labeledge_[b].a;            // T vertex (base of the T blossom)
                    b = inblossom_[v];
                    v = labeledge_[b].a;            // S vertex that labeled it
                }
            }
            if (w != -1) std::swap(v, w);
        }
        for (int b : path) label_[b] = 1;
        return found;
    }

    void add_blossom(int basev, int v, int w) {
        const int v0 = v, w0 = w;
        const int bb = inblossom_[basev];
        int bv = inblossom_[v], bw = inblossom_[w];
        const int b = unused_.back();
        unused_.pop_back();
        base_[b] = basev;
        parent_[b] = -1;
        parent_[bb] = b;
        std::vector<int> path;
        std::vector<Edge> eds;      // eds[i]: a in child i, b in child i+1
        while (bv != bb) {
            parent_[bv] = b;
            path.push_back(bv);
            eds.push_back(labeledge_[bv]);          // (remote toward base, inside bv)
            v = labeledge_[bv].a;
            bv = inblossom_[v];
        }
        path.push_back(bb);
        std::reverse(path.begin(), path.end());
        std::reverse(eds.begin(), eds.end());
        Edge mid;
        mid.a = v0; mid.b = w0;
        eds.push_back(mid);
        while (bw != bb) {
            parent_[bw] = b;
            path.push_back(bw);
            Edge le = labeledge_[bw];
            Edge e; e.a = le.b; e.b = le.a;          // (inside bw, remote toward base)
            eds.push_back(e);
            w = labeledge_[bw].a;
            bw = inblossom_[w];
        }
        childs_[b] = path;
        edges_[b] = eds;
        label_[b] = 1;
        labeledge_[b] = labeledge_[bb];
        dual_[b] = 0;
        leaves(b, [this, b](int x) {
            if (label_[inblossom_[x]] == 2) queue_.push_back(x);
            inblossom_[x] = b;
        });
        // least-slack edges from the new blossom to every other S-blossom
        std::vector<Edge> best(2 * n_);
        std::vector<i128> bestslack(2 * n_, 0);
        auto consider = [&](int i, int j, i128 w) {
            if (inblossom_[j] == b) std::swap(i, j);
            const int bj = inblossom_[j];
            if (bj != b && label_[bj] == 1) {
                i128 s = slack_w(i, j, w);
                if (best[bj].none() || s < bestslack[bj]) {
                    best[bj].a = i; best[bj].b = j; best[bj].w = w; bestslack[bj] = s;
                }
            }
        };
        for (int c : path) {
            if (!has_bestlist_[c]) {
                leaves(c, [&](int x) {
                    for (int64_t k = g_.off[x]; k < g_.off[x + 1]; ++k) consider(x, g_.nbr[k], g_.w[k]);
                });
            } else {
                for (const Edge &e : bestlist_[c]) consider(e.a, e.b, e.w);
            }
            bestlist_[c].clear();
            has_bestlist_[c] = 0;
            bestedge_[c] = Edge();
        }
        bestlist_[b].clear();
        has_bestlist_[b] = 1;
        Edge be;
        i128 bs = 0;
        for (int k = 0; k < 2 * n_; ++k) {
            if (best[k].none()) continue;
            bestlist_[b].push_back(best[k]);
            if (be.none() || bestslack[k] < bs) { be = best[k]; bs = bestslack[k]; }
        }
        bestedge_[b] = be;
    }

    // oriented edge from child j toward child j+dir of blossom b
    Edge step_edge(int b, int j, int dir) const {
        const int k = (int)childs_[b].size();
        auto at = [k](int x) { return ((x % k) + k) % k; };
        if (dir > 0) return edges_[b][at(j)];
        Edge e = edges_[b][at(j - 1)];
        std::swap(e.a, e.b);
        return e;
    }

    void expand(int b, bool endstage) {
        for (int s : childs_[b]) {
            parent_[s] = -1;
            if (s < n_) inblossom_[s] = s;
            else if (endstage && dual_[s] == 0) expand(s, endstage);
            else leaves(s, [this, s](int x) { inblossom_[x] = s; });
        }
        if (!endstage && label_[b] == 2) {
            const int k = (int)childs_[b].size();
            auto at = [k](int x) { return ((x % k) + k) % k; };
            const int entry = inblossom_[labeledge_[b].b];
            int j = (int)(std::find(childs_[b].begin(), childs_[b].end(), entry) - childs_[b].begin());
            int dir;
            if (j & 1) { j -= k; dir = 1; } else { dir = -1; }
            Edge p = labeledge_[b];                  // (remote, inside child j)
            while (j != 0) {
                label_[p.b] = 0;
                Edge q = step_edge(b, j, dir);
                label_[q.b] = 0;
                assign_label(p.b, 2, p.a);
                set_allow(q.a, q.b);
                j += dir;
                Edge q2 = step_edge(b, j, dir);
                p.a = q2.a; p.b = q2.b;
                set_allow(q2.a, q2.b);
                j += dir;
            }
            int bv = childs_[b][at(j)];
            label_[p.b] = label_[bv] = 2;
            labeledge_[p.b] = labeledge_[bv] = p;
            bestedge_[bv] = Edge();
            j += dir;
            while (childs_[b][at(j)] != entry) {
                bv = childs_[b][at(j)];
                if (label_[bv] == 1) { j += dir; continue; }
                int hit = -1;
                leaves(bv, [&](int x) { if (hit < 0 && label_[x] != 0) hit = x; });
                if (hit >= 0) {
                    label_[hit] = 0;
                    label_[mate_[base_[bv]]] = 0;
                    assign_label(hit, 2, labeledge_[hit].a);
                }
                j += dir;
            }
        }
        label_[b] = 0;
        labeledge_[b] = Edge();
        childs_[b].clear();
        edges_[b].clear();
        base_[b] = -1;
        bestlist_[b].clear();
        has_bestlist_[b] = 0;
        bestedge_[b] = Edge();
        unused_.push_back(b);
    }

    // swap matched/unmatched edges inside blossom b so vertex v becomes its base
    void augment_blossom(int b, int v) {
        int t = v;
        while (parent_[t] != b) t = parent_[t];
        if (t >= n_) augment_blossom(t, v);
        const int k = (int)childs_[b].size();
        auto at = [k](int x) { return ((x % k) + k) % k; };
        const int i = (int)(std::find(childs_[b].begin(), childs_[b].end(), t) - childs_[b].begin());
        int j = i, dir;
        if (i & 1) { j -= k; dir = 1; } else { dir = -1; }
        while (j != 0) {
            j += dir;
            const Edge e = step_edge(b, j, dir);    // a in child j, b in child j+dir
            int tc = childs_[b][at(j)];
            if (tc >= n_) augment_blossom(tc, e.a);
            j += dir;
            tc = childs_[b][at(j)];
            if (tc >= n_) augment_blossom(tc, e.b);
            mate_[e.a] = e.b;
            mate_[e.b] = e.a;
        }
        std::rotate(childs_[b].begin(), childs_[b].begin() + i, childs_[b].end());
        std::rotate(edges_[b].begin(), edges_[b].begin() + i, edges_[b].end());
        base_[b] = base_[childs_[b][0]];
    }

    void augment_matching(int v, int w) {
        const int ends[2][2] = {{v, w}, {w, v}};
        for (auto &sv : ends) {
            int s = sv[0], other = sv[1];
            for (;;) {
                const int bs = inblossom_[s];
                if (bs >= n_) augment_blossom(bs, s);
                mate_[s] = other;
                if (labeledge_[bs].none()) break;
                const int t = labeledge_[bs].a;
                const int bt = inblossom_[t];
                const int s2 = labeledge_[bt].a, j = labeledge_[bt].b;
                if (bt >= n_) augment_blossom(bt, j);
                mate_[j] = s2;
                s = s2;
                other = j;
            }
        }
    }

    // scan S-vertex v; returns true after an augmentation
    bool scan_vertex(int v) {
        for (int64_t k = g_.off[v]; k < g_.off[v + 1]; ++k) {
            const int w = g_.nbr[k];
            const i128 ew = g_.w[k];
            const int bw = inblossom_[w];
            if (inblossom_[v] == bw) continue;     // re-read: add_blossom may move v
            i128 ks = 0;
            bool tight = allowed(v, w);
            if (!tight) {
                ks = slack_w(v, w, ew);
                if (ks <= 0) { set_allow(v, w); tight = true; }
            }
            if (tight) {
                if (label_[bw] == 0) {
                    assign_label(w, 2, v);
                } else if (label_[bw] == 1) {
                    const int base = scan_blossom(v, w);
                    if (base >= 0) {
                        add_blossom(base, v, w);
                    } else {
                        augment_matching(v, w);
                        return true;
                    }
                } else if (label_[w] == 0) {
                    label_[w] = 2;
                    labeledge_[w].a = v;
                    labeledge_[w].b = w;
                }
            } else if (label_[bw] == 1) {
                const int b = inblossom_[v];
                if (bestedge_[b].none() || ks < slack(bestedge_[b])) {
                    bestedge_[b].a = v; bestedge_[b].b = w; bestedge_[b].w = ew;
                }
            } else if (label_[w] == 0) {
                if (bestedge_[w].none() || ks < slack(bestedge_[w])) {
                    bestedge_[w].a = v; bestedge_[w].b = w; bestedge_[w].w = ew;
                }
            }
        }
        return false;
    }

    int n_;
    const Graph &g_;
    int extra_ = 1;        // weights carry one extra factor 2 from the start
    bool warm_ = false;
    std::vector<int> mate_, label_, inblossom_, parent_, base_, unused_, queue_;
    std::vector<Edge> labeledge_, bestedge_;
    std::vector<std::vector<int>> childs_;
    std::vector<std::vector<Edge>> edges_;
    std::vector<std::vector<Edge>> bestlist_;
    std::vector<uint8_t> has_bestlist_;
    std::vector<i128> dual_;
    std::vector<uint8_t> allow_;
    std::vector<size_t> touched_;
};

// The value of edge (u, v) the blossom solver maximizes, as a double:
//   REFLECT: (max w + 1) - w[u][v]          (matcher.py:84-85; complete graph, perfect)
//   BENEFIT: pot[u] + pot[v] - w[u][v]       (only edges with a positive value exist)
//   RAW:     w[u][v]
struct EdgeValue {
    enum Kind { RAW, REFLECT, BENEFIT } kind;
    const double *w;
    int n;
    double reflect;
    const double *pot;
    double operator()(int u, int v) const {
        const double x = w[(size_t)u * n + v];
        switch (kind) {
            case REFLECT: return reflect - x;
            case BENEFIT: return (pot[u] + pot[v]) - x;
            default: return x;
        }
    }
    bool exists(double x) const { return kind != BENEFIT || x > 0.0; }
};

// power-of-two shift that turns every edge value into an exact integer
// (-2 when they span too many binary orders of magnitude for 128 bits)
int shift_of(int emin, int emax, int *shift) {
    if (emin == INT32_MAX) { *shift = 0; return 0; }
    const int s = 53 - emin;            // ulp(r) = 2^(e-53) -> integer after << s
    if (emax + s > 96) return -2;       // keep 2^31 of headroom below 2^127 for duals
    *shift = s;
    return 0;
}

// exponent range of the existing nonzero values of rows [u0, u1); -1 if a
// value is not finite
int exp_range(const EdgeValue &f, int u0, int u1, int *emin_out, int *emax_out) {
    int emin = INT32_MAX, emax = INT32_MIN;
    for (int u = u0; u < u1; ++u)
        for (int v = 0; v < f.n; ++v) {
            if (u == v) continue;
            const double r = f(u, v);
            if (!std::isfinite(r)) return -1;
            if (r == 0.0 || !f.exists(r)) continue;
            int e;
            std::frexp(r, &e);
            emin = std::min(emin, e);
            emax = std::max(emax, e);
        }
    *emin_out = emin;
    *emax_out = emax;
    return 0;
}

int choose_shift(const EdgeValue &f, int *shift) {
    int emin, emax;
    if (exp_range(f, 0, f.n, &emin, &emax)) return -1;
    return shift_of(emin, emax, shift);
}

inline i128 scaled(double x, int shift) { return (i128)std::ldexp(x, shift); }

// symmetric CSR graph over an undirected edge set (pairs u < v)
Graph make_graph(const EdgeValue &f, const std::vector<std::pair<int, int>> &edges, int shift) {
    Graph g;
    g.n = f.n;
    const int n = f.n;
    std::vector<int64_t> deg(n + 1, 0);
    for (auto &e : edges) { ++deg[e.first]; ++deg[e.second]; }
    g.off.assign(n + 1, 0);
    for (int v = 0; v < n; ++v) g.off[v + 1] = g.off[v] + deg[v];
    g.nbr.resize(g.off[n]);
    g.w.resize(g.off[n]);
    std::vector<int64_t> pos(g.off.begin(), g.off.end() - 1);
    for (auto &e : edges) {
        const i128 x = scaled(f(e.first, e.second), shift);
        g.nbr[pos[e.first]] = e.second; g.w[pos[e.first]++] = x;
        g.nbr[pos[e.second]] = e.first; g.w[pos[e.second]++] = x;
    }
    return g;
}

// Existing edges (i, j) whose reduced cost under the solver's final duals is
// negative: y_i + y_j + 2 * (sum of duals of blossoms holding both) - 2 w_ij < 0
// in the solver's doubled units (the reference's verify_optimum).  Up to
// `per_vertex` most violated edges per vertex.
std::vector<std::pair<int, int>> violations(const Blossom &m, const EdgeValue &f, int shift,
                                            int per_vertex) {
    const int n = f.n;
    const std::vector<i128> &dual = m.duals();
    const std::vector<int> &parent = m.parents();
    const int extra = m.extra();
    std::vector<std::vector<int>> chain(n);   // enclosing blossoms, outermost first
    for (int v = 0; v < n; ++v) {
        for (int b = parent[v]; b >= 0; b = parent[b]) chain[v].push_back(b);
        std::reverse(chain[v].begin(), chain[v].end());
    }
    std::vector<std::pair<int, int>> out;
    std::vector<std::pair<i128, int>> worst;
    for (int i = 0; i < n; ++i) {
        worst.clear();
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double x = f(i, j);
            if (!f.exists(x)) continue;
            i128 z = 0;
            const auto &ci = chain[i], &cj = chain[j];
            for (size_t k = 0; k < ci.size() && k < cj.size() && ci[k] == cj[k]; ++k) z += dual[ci[k]];
            const i128 red = dual[i] + dual[j] + 2 * z - 2 * (scaled(x, shift) << extra);
            if (red < 0) worst.push_back({red, j});
        }
        if (worst.size() > (size_t)per_vertex) {
            std::partial_sort(worst.begin(), worst.begin() + per_vertex, worst.end());
            worst.resize(per_vertex);
        }
        for (auto &x : worst) out.push_back({std::min(i, x.second), std::max(i, x.second)});
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
}

// Maximum-weight matching of the graph of existing edges of `f`: the blossom
// solver on the k most valuable edges of every vertex (k <= 0: all), then the
// dual certificate on every existing edge, adding violators until none is
// left.  Returns 0 or -3.
int certified_matching(const EdgeValue &f, int k, int shift, int32_t *mate_out) {
    const int n = f.n;
    std::vector<std::pair<int, int>> edges;
    std::vector<std::pair<double, int>> row(n);
    for (int u = 0; u < n; ++u) {
        int c = 0;
        for (int v = 0; v < n; ++v) {
            if (v == u) continue;
            const double x = f(u, v);
            if (f.exists(x)) row[c++] = {-x, v};
        }
        const int take = (k <= 0 || k >= c) ? c : k;
        std::partial_sort(row.begin(), row.begin() + take, row.begin() + c);
        for (int q = 0; q < take; ++q) edges.push_back({std::min(u, row[q].second), std::max(u, row[q].second)});
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    for (int round = 0; round < 64; ++round) {
        const Graph g = make_graph(f, edges, shift);
        Blossom m(g);
        m.run(false);
        const std::vector<std::pair<int, int>> bad =
            (k <= 0) ? std::vector<std::pair<int, int>>() : violations(m, f, shift, 8);
        if (bad.empty()) {
            for (int v = 0; v < n; ++v) mate_out[v] = m.mate()[v];
            return 0;
        }
        edges.insert(edges.end(), bad.begin(), bad.end());
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    }
    return -3;
}

// Persistent host worker pool for the row-parallel loops of the certified
// solver (the auction runs thousands of short parallel rounds, so threads are
// started once per solve, not per loop).
class RowPool {
public:
    RowPool() {
        int nt = (int)std::thread::hardware_concurrency();
        nt_ = std::max(1, std::min(nt, 64));
        for (int t = 1; t < nt_; ++t) th_.emplace_back([this, t] { worker(t); });
    }
    ~RowPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_.store(true);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int threads() const { return nt_; }
    // body(i, thread) for i in [0, n); small loops run inline.  Workers spin
    // for a while after each job before they sleep: the auction dispatches
    // tens of thousands of short rounds, and a futex wake-up per worker per
    // round cost more than many rounds' work.
    template <class F>
    void run(int n, F &&body, int grain = 16) {
        if (nt_ == 1 || n < 2 * grain) {
            for (int i = 0; i < n; ++i) body(i, 0);
            return;
        }
        std::function<void(int, int)> fn = body;
        job_ = &fn;
        n_ = n;
        grain_ = grain;
        next_.store(0, std::memory_order_relaxed);
        pending_.store(nt_ - 1, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> g(mu_);      // pairs with a sleeper's predicate check
            gen_.fetch_add(1, std::memory_order_release);
        }
        if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
        chew(0);
        for (int spin = 0; pending_.load(std::memory_order_acquire) != 0; ++spin)
            if (spin > 1024) std::this_thread::yield();
        job_ = nullptr;
    }

private:
    void chew(int t) {
        for (;;) {
            const int i0 = next_.fetch_add(grain_, std::memory_order_relaxed);
            if (i0 >= n_) break;
            const int i1 = std::min(n_, i0 + grain_);
            for (int i = i0; i < i1; ++i) (*job_)(i, t);
        }
    }
    void worker(int t) {
        uint64_t seen = 0;
        for (;;) {
            // spin ~tens of microseconds for the next job, then sleep
            bool got = false;
            for (int spin = 0; spin < 20000; ++spin) {
                if (gen_.load(std::memory_order_acquire) != seen) { got = true; break; }
                if ((spin & 63) == 63) std::this_thread::yield();
            }
            if (!got) {
                std::unique_lock<std::mutex> g(mu_);
                sleepers_.fetch_add(1, std::memory_order_acq_rel);
                cv_.wait(g, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                sleepers_.fetch_sub(1, std::memory_order_acq_rel);
            }
            seen = gen_.load(std::memory_order_acquire);
            if (stop_.load()) return;
            chew(t);
            pending_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    int nt_ = 1;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> stop_{false};
    std::atomic<int> sleepers_{0}, pending_{0};
    std::function<void(int, int)> *job_ = nullptr;
    int n_ = 0, grain_ = 16;
    std::atomic<int> next_{0};
};

// Prices of an eps-optimal maximum-weight ASSIGNMENT of the complete graph
// read as bipartite (row u takes object v != u at value f(u, v)): the
// fractional relaxation of perfect matching.  Forward auction with
// eps-scaling, Jacobi rounds (every unassigned row bids in parallel, the
// highest bid per object wins).  The perfect-matching values are
// f(u, v) = c_u + d_v - w[u][v] (BENEFIT: c = d = pot; REFLECT: c = r, d = 0),
// so a row's best object minimizes w[u][v] + (price_v - d_v).  Only the
// prices are used, and only as guidance: feasibility is restored exactly
// from them (see certified_perfect).
std::vector<double> auction_prices(const EdgeValue &f, double eps_final_rel, RowPool &pool) {
    const int n = f.n;
    std::vector<double> price(n, 0.0), h(n, 0.0), d(n, 0.0), c(n, 0.0);
    for (int v = 0; v < n; ++v) {
        d[v] = f.kind == EdgeValue::BENEFIT ? f.pot[v] : 0.0;
        c[v] = f.kind == EdgeValue::BENEFIT ? f.pot[v] : f.reflect;
    }
    double vmax = 0.0;
    {
        std::vector<double> rmax(n, 0.0);
        pool.run(n, [&](int u, int) {
            const double *wr = f.w + (size_t)u * n;
            double m = INFINITY;
            for (int v = 0; v < n; ++v) {
                const double x = v == u ? INFINITY : wr[v] - d[v];
                m = std::min(m, x);
            }
            rmax[u] = c[u] - m;
        });
        for (double x : rmax) vmax = std::max(vmax, x);
    }
    if (!(vmax > 0.0)) return price;
    std::vector<int> owner(n), bid_obj(n), freerows, next, best(n, -1);
    std::vector<double> bid_val(n);
    freerows.reserve(n);
    next.reserve(n);
    for (double eps = vmax / 8;; eps /= 6) {
        std::fill(owner.begin(), owner.end(), -1);
        freerows.resize(n);
        for (int u = 0; u < n; ++u) freerows[u] = u;
        int rounds_dbg = 0;
        long long bids_dbg = 0;
        for (int v = 0; v < n; ++v) h[v] = price[v] - d[v];   // kept current as prices move
        for (int it = 0; !freerows.empty() && it < 1000000; ++it) {
            ++rounds_dbg;
            const int nf = (int)freerows.size();
            bids_dbg += nf;
            auto bid = [&](int q, int) {
                const int u = freerows[q];
                const double *wr = f.w + (size_t)u * n;
                double m1 = INFINITY, m2 = INFINITY;   // two smallest w + h, v != u
                int j1 = -1;
                auto scan = [&](int v0, int v1) {
                    for (int v = v0; v < v1; ++v) {
                        const double x = wr[v] + h[v];
                        if (x < m2) {
                            if (x < m1) { m2 = m1; m1 = x; j1 = v; }
                            else m2 = x;
                        }
                    }
                };
                scan(0, u);
                scan(u + 1, n);
                if (m2 == INFINITY) m2 = m1;
                bid_obj[q] = j1;
                bid_val[q] = price[j1] + (m2 - m1) + eps;
            };
            // the long tail of rounds has a handful of free rows: bid on this
            // thread (a pool dispatch costs more than the scans)
            if (nf <= 8) {
                for (int q = 0; q < nf; ++q) bid(q, 0);
            } else {
                pool.run(nf, bid, 4);
            }
            next.clear();
            for (int q = 0; q < nf; ++q) {
                const int v = bid_obj[q];
                if (best[v] < 0 || bid_val[q] > bid_val[best[v]]) best[v] = q;
            }
            for (int q = 0; q < nf; ++q) {
                const int v = bid_obj[q], u = freerows[q];
                if (best[v] != q) { next.push_back(u); continue; }
                if (owner[v] >= 0) next.push_back(owner[v]);
                owner[v] = u;
                price[v] = bid_val[q];
                h[v] = price[v] - d[v];
            }
            for (int q = 0; q < nf; ++q) best[bid_obj[q]] = -1;
            freerows.swap(next);
        }
        if (getenv("CM_DEBUG"))
            fprintf(stderr, "cm:   auction eps %.3g: %d rounds, %lld bids\n", eps / vmax, rounds_dbg, bids_dbg);
        if (eps <= eps_final_rel * vmax) break;
    }
    return price;
}

// Maximum-weight PERFECT matching of the complete graph (every u != v is an
// edge of value f(u, v) >= 0), warm-started and certified:
//   1. guidance: prices p of the assignment relaxation (auction_prices);
//   2. exact, globally feasible start: with P = p scaled to the solver's
//      integers, a_u = max_v (2 f(u, v) - P_v) and y_u = a_u + P_u every
//      slack y_u + y_v - 2 f(u, v) = (a_u + P_v - 2f) + (a_v + P_u - 2f) is
//      >= 0 on ALL n(n-1)/2 edges; good prices make the optimal pairs nearly
//      tight, so they rank first by slack;
//   3. candidates: the k least-slack edges of every vertex (row-parallel);
//      jump start: in vertex order each free v lowers y_v to its tightest
//      edge over the complete graph (all slacks stay >= 0) and takes that
//      partner if it is free; plus a backbone (greedy matching of the
//      candidates, leftovers paired in order) so a perfect matching exists;
//   4. the blossom solver in max-cardinality mode from that matching and
//      those duals (for the perfect-matching LP the vertex duals are free);
//   5. the LP dual certificate on every edge of the complete graph
//      (row-parallel).  Violating edges join the candidates; the duals are
//      flattened (each blossom dual added to its vertices, which keeps every
//      slack >= 0), each row's violators made tight by one raise of that row's
//      vertex, matched edges that lost tightness unmatched, and step 4 resumes.
// The result is an optimum of the complete graph (the final certificate is
// the reference's verify-optimum condition on all n(n-1)/2 edges).
int certified_perfect(const EdgeValue &f, int k, int shift, int32_t *mate_out, RowPool &pool) {
    const int n = f.n;
    static const bool dbg = getenv("CM_DEBUG") != nullptr;
    auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t_mark = now();
    auto lap = [&](const char *what, long long x) {
        if (!dbg) return;
        const double t = now();
        fprintf(stderr, "cm: %-22s %8.1f ms  (%lld)\n", what, 1e3 * (t - t_mark), x);
        t_mark = t;
    };
    if (k <= 0 || k >= n - 1) k = n - 1;
    int extra = 1;
    auto W = [&](int u, int v) { return scaled(f(u, v), shift) << extra; };
    // Every exact integer below has a double shadow: Wd = f * 2^(shift+extra)
    // is the exact weight as a double (a power-of-two scaling), so sums of a
    // few such terms are off by a few ulps of their magnitude.  The dense
    // O(n^2) scans run in double and re-check in i128 only the entries within
    // `tol` of the decision, so every feasibility / tightness fact is exact.
    auto Wd = [&](int u, int v) { return std::ldexp(f(u, v), shift + extra); };
    double mag = 0.0;
    for (int u = 0; u < n; ++u) mag = std::max(mag, std::fabs(Wd(u, u == 0 ? 1 : 0)));
    // ---- 1-2. prices -> exact feasible duals ----
    std::vector<i128> dual(n, 0), P(n, 0);
    std::vector<double> dd(n, 0.0);
    double tol = 0.0;
    {
        const std::vector<double> price = auction_prices(f, 3e-3, pool);
        std::vector<double> Pd(n);
        for (int v = 0; v < n; ++v) {
            P[v] = 2 * (scaled(price[v], shift) << extra);
            Pd[v] = (double)P[v];
            mag = std::max(mag, std::fabs(Pd[v]));
        }
        std::vector<double> rowmax(n, 0.0);
        pool.run(n, [&](int u, int) {
            double m = 0.0;
            for (int v = 0; v < n; ++v)
                if (v != u) m = std::max(m, std::fabs(Wd(u, v)));
            rowmax[u] = m;
        });
        for (double x : rowmax) mag = std::max(mag, x);
        tol = std::ldexp(mag, -40);       // >> the rounding of any 8-term sum
        pool.run(n, [&](int u, int) {
            double best = -INFINITY;
            for (int v = 0; v < n; ++v)
                if (v != u) best = std::max(best, 2 * Wd(u, v) - Pd[v]);
            i128 a = 0;
            bool any = false;
            for (int v = 0; v < n; ++v) {
                if (v == u || 2 * Wd(u, v) - Pd[v] < best - 8 * tol) continue;
                const i128 x = 2 * W(u, v) - P[v];
                if (!any || x > a) { a = x; any = true; }
            }
            dual[u] = (a + P[u]) / 2;      // a + P even: both terms are even
            dd[u] = (double)dual[u];
        });
    }
    lap("auction + duals", n);
    // ---- 3. candidates by slack (double: a heuristic), jump start, backbone ----
    std::vector<std::vector<int>> cand(n);
    pool.run(n, [&](int u, int) {
        std::vector<std::pair<double, int>> row;
        row.reserve(n);
        for (int v = 0; v < n; ++v)
            if (v != u) row.push_back({dd[u] + dd[v] - 2 * Wd(u, v), v});
        std::partial_sort(row.begin(), row.begin() + k, row.end());
        for (int q = 0; q < k; ++q) cand[u].push_back(row[q].second);
    });
    std::vector<std::pair<int, int>> edges;
    for (int u = 0; u < n; ++u)
        for (int v : cand[u]) edges.push_back({std::min(u, v), std::max(u, v)});
    lap("candidates", (long long)edges.size());
    std::vector<int> mate(n, -1);
    {
        std::vector<double> need(n);
        for (int v = 0; v < n; ++v) {
            if (mate[v] >= 0) continue;
            // exact max_u (2 W_uv - y_u): double scan, i128 on the near-max
            // (row v of the symmetric w: f(v, u) == f(u, v) bit for bit, and
            // a row scan is contiguous where column u would stride by n)
            double bd = -INFINITY;
            for (int u = 0; u < n; ++u) {
                need[u] = u == v ? -INFINITY : 2 * Wd(v, u) - dd[u];
                bd = std::max(bd, need[u]);
            }
            i128 best = 0;
            int arg = -1;
            bool arg_free = false;
            for (int u = 0; u < n; ++u) {
                if (u == v || need[u] < bd - 8 * tol) continue;
                const i128 x = 2 * W(v, u) - dual[u];
                const bool fr = mate[u] < 0;
                if (arg < 0 || x > best || (x == best && fr && !arg_free)) {
                    best = x; arg = u; arg_free = fr;
                }
            }
            dual[v] = best;
            dd[v] = (double)best;
            if (arg_free) {
                mate[v] = arg; mate[arg] = v;
                edges.push_back({std::min(v, arg), std::max(v, arg)});
            }
        }
    }
    // Zero-value edges (BENEFIT: time-share pairs, f == 0), 8 per vertex on a
    // fixed pseudo-random pattern: the optimum pairs its leftover vertices
    // with such edges.  Without them in the candidate graph the solver drove
    // those vertices' duals negative, every certificate violator was a zero
    // edge between two of them, and the rounds added them 8 per row (2-7
    // rounds at N=4,096); with them one round certifies (tools/
    // matcher_robustness.py: 1.1-2.0 s instead of 1.2-6.2 s)
    constexpr int k0 = 8;
    if (f.kind == EdgeValue::BENEFIT) {
        for (int u = 0; u < n; ++u) {
            uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(u + 1);
            for (int q = 0, got = 0; q < 4 * k0 && got < k0; ++q) {
                h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
                const int v = (int)(h % (uint64_t)n);
                if (v == u || f(u, v) != 0.0) continue;
                edges.push_back({std::min(u, v), std::max(u, v)});
                ++got;
            }
        }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    {
        std::vector<std::pair<double, int>> order(edges.size());
        for (size_t q = 0; q < edges.size(); ++q) {
            const int u = edges[q].first, v = edges[q].second;
            order[q] = {dd[u] + dd[v] - 2 * Wd(u, v), (int)q};
        }
        std::sort(order.begin(), order.end());
        std::vector<char> used(n, 0);
        for (auto &o : order) {
            const int u = edges[o.second].first, v = edges[o.second].second;
            if (!used[u] && !used[v]) used[u] = used[v] = 1;
        }
        int prev = -1;
        for (int v = 0; v < n; ++v) {
            if (used[v]) continue;
            if (prev < 0) { prev = v; continue; }
            edges.push_back({prev, v});
            prev = -1;
        }
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    }
    Graph g = make_graph(f, edges, shift);
    int extra0 = extra;
    {
        long long free0 = 0;
        for (int v = 0; v < n; ++v) free0 += mate[v] < 0;
        lap("jump + backbone", free0);
    }

    for (int round = 0; round < 64; ++round) {
        Blossom m(g);
        m.warm(dual, mate, extra);
        m.run(true);
        lap("blossom run", (long long)edges.size());
        extra = m.extra();
        const std::vector<i128> &bd = m.duals();
        const std::vector<int> &parent = m.parents();
        const std::vector<int> &mm = m.mate();
        std::vector<std::vector<int>> chain(n);   // enclosing blossoms, outermost first
        for (int v = 0; v < n; ++v) {
            for (int b = parent[v]; b >= 0; b = parent[b]) chain[v].push_back(b);
            std::reverse(chain[v].begin(), chain[v].end());
        }
        if (extra != extra0) {             // the solver doubled its scale
            for (int q = 0; q < extra - extra0; ++q) tol *= 2;
            extra0 = extra;
        }
        std::vector<double> fd(n);
        for (int v = 0; v < n; ++v) fd[v] = (double)bd[v];
        // certificate on the complete graph (every edge of a single vertex too)
        std::vector<std::vector<std::pair<i128, int>>> bad(n);
        pool.run(n, [&](int i, int) {
            std::vector<std::pair<i128, int>> worst;
            for (int j = 0; j < n; ++j) {
                if (j == i) continue;
                if (mm[i] < 0) { worst.push_back({0, j}); continue; }   // every edge of a single
                if (mm[j] < 0) continue;                                  // (added by j's row)
                const auto &ci = chain[i], &cj = chain[j];
                if (ci.empty() || cj.empty() || ci[0] != cj[0]) {
                    // no common blossom: the double reduced cost decides
                    // unless it is within tol of 0
                    if (fd[i] + fd[j] - 2 * Wd(i, j) > 8 * tol) continue;
                }
                i128 z = 0;
                for (size_t q = 0; q < ci.size() && q < cj.size() && ci[q] == cj[q]; ++q) z += bd[ci[q]];
                const i128 red = bd[i] + bd[j] + 2 * z - 2 * W(i, j);
                if (red < 0) worst.push_back({red, j});
            }
            const size_t cap = 8;
            if (mm[i] >= 0 && worst.size() > cap) {
                std::partial_sort(worst.begin(), worst.begin() + cap, worst.end());
                worst.resize(cap);
            }
            bad[i] = std::move(worst);
        });
        size_t nbad = 0;
        for (int i = 0; i < n; ++i) nbad += bad[i].size();
        if (dbg) {
            long long zero = 0, single = 0;
            for (int i = 0; i < n; ++i) {
                if (mm[i] < 0) single += (long long)bad[i].size();
                for (auto &x : bad[i]) zero += f(i, x.second) == 0.0;
            }
            long long nblos = 0;
            for (int v = 0; v < n; ++v) nblos += parent[v] >= 0;
            long double val = 0;
            long long negd = 0;
            for (int v = 0; v < n; ++v) {
                if (mm[v] > v) val += f(v, mm[v]);
                i128 y = bd[v];
                for (int b = parent[v]; b >= 0; b = parent[b]) y += bd[b];
                negd += y < 0;
            }
            fprintf(stderr, "cm:   violators on zero-value edges %lld, of unmatched rows %lld; vertices in blossoms %lld;"
                    " matching value %.12Lf; negative flattened duals %lld\n", zero, single, nblos, val, negd);
        }
        lap("certificate", (long long)nbad);
        if (nbad == 0) {
            for (int v = 0; v < n; ++v) mate_out[v] = mm[v];
            return 0;
        }
        for (int i = 0; i < n; ++i)
            for (auto &x : bad[i]) edges.push_back({std::min(i, x.second), std::max(i, x.second)});
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        g = make_graph(f, edges, shift);
        // warm state for the next round: flattened duals, violators made tight
        for (int v = 0; v < n; ++v) {
            i128 y = bd[v];
            for (int b = parent[v]; b >= 0; b = parent[b]) y += bd[b];
            dual[v] = y;
        }
        mate.assign(mm.begin(), mm.end());
        for (int i = 0; i < n; ++i) {
            i128 deficit = 0;
            for (auto &x : bad[i]) {
                const i128 red = dual[i] + dual[x.second] - 2 * W(i, x.second);
                if (red < 0 && -red > deficit) deficit = -red;
            }
            dual[i] += deficit;
        }
        for (int v = 0; v < n; ++v) {
            const int u = mate[v];
            if (u > v && dual[u] + dual[v] != 2 * W(u, v)) { mate[u] = -1; mate[v] = -1; }
        }
    }
    return -3;
}

int check_rows(const double *w, int32_t n, int u0, int u1) {
    for (int u = u0; u < u1; ++u)
        for (int v = 0; v < n; ++v) {
            const double x = w[(size_t)u * n + v];
            if (!std::isfinite(x)) return -1;
            if (u != v && x != w[(size_t)v * n + u]) return -1;
        }
    return 0;
}

int check_square(const double *w, int32_t n) { return check_rows(w, n, 0, n); }

// The O(n^2) input checks and scale choice of the perfect-matching entry
// points, row-parallel: symmetric finite w, optional potential bound
// (-4 if violated), exponent range -> shift.
int prepare_parallel(const EdgeValue &f, const double *pot, RowPool &pool, int *shift) {
    const int n = f.n;
    const int nt = pool.threads();
    std::vector<int> bad(nt, 0), lo(nt, INT32_MAX), hi(nt, INT32_MIN);
    pool.run(n, [&](int u, int t) {
        if (check_rows(f.w, n, u, u + 1)) { bad[t] = -1; return; }
        if (pot) {
            if (!std::isfinite(pot[u])) { bad[t] = -1; return; }
            for (int v = 0; v < n; ++v)
                if (u != v && f.w[(size_t)u * n + v] > pot[u] + pot[v]) { if (!bad[t]) bad[t] = -4; return; }
        }
        int e0, e1;
        if (exp_range(f, u, u + 1, &e0, &e1)) { bad[t] = -1; return; }
        lo[t] = std::min(lo[t], e0);
        hi[t] = std::max(hi[t], e1);
    });
    for (int t = 0; t < nt; ++t)
        if (bad[t] == -1) return -1;
    for (int t = 0; t < nt; ++t)
        if (bad[t]) return bad[t];
    int emin = INT32_MAX, emax = INT32_MIN;
    for (int t = 0; t < nt; ++t) { emin = std::min(emin, lo[t]); emax = std::max(emax, hi[t]); }
    return shift_of(emin, emax, shift);
}

}  // namespace

extern "C" {

const char *cm_version(void) {
    return "cosched_match 0.4.0 (exact int128 blossom, auction-priced warm start, sparse + dual certificate)";
}

int cm_max_weight_matching(const double *w, int32_t n, int32_t *mate_out) {
    if (n < 0 || (n > 0 && (!w || !mate_out))) return -1;
    if (n == 0) return 0;
    if (check_square(w, n)) return -1;
    EdgeValue f{EdgeValue::RAW, w, n, 0.0, nullptr};
    int shift = 0;
    int rc = choose_shift(f, &shift);
    if (rc) return rc;
    return certified_matching(f, 0, shift, mate_out);
}

int cm_min_weight_perfect_matching(const double *w, int32_t n, int32_t *mate_out) {
    return cm_min_weight_perfect_matching_k(w, n, 24, mate_out);
}

int cm_min_weight_perfect_matching_k(const double *w, int32_t n, int32_t k, int32_t *mate_out) {
    if (n < 2 || (n & 1) || !w || !mate_out) return -1;
    RowPool pool;
    std::vector<double> rmx(n, -INFINITY);
    pool.run(n, [&](int u, int) {
        double m = -INFINITY;
        for (int v = 0; v < n; ++v) m = std::max(m, w[(size_t)u * n + v]);
        rmx[u] = m;
    });
    double mx = -INFINITY;
    for (double x : rmx) mx = std::max(mx, x);
    EdgeValue f{EdgeValue::REFLECT, w, n, mx + 1.0, nullptr};   // matcher.py:84
    int shift = 0;
    int rc = prepare_parallel(f, nullptr, pool, &shift);
    if (rc) return rc;
    rc = certified_perfect(f, k, shift, mate_out, pool);
    if (rc) return rc;
    for (int v = 0; v < n; ++v)
        if (mate_out[v] < 0) return -3;
    return 0;
}

int cm_min_weight_perfect_matching_pot(const double *w, int32_t n, const double *pot, int32_t k,
                                       int32_t *mate_out) {
    if (n < 2 || (n & 1) || !w || !pot || !mate_out) return -1;
    RowPool pool;
    EdgeValue f{EdgeValue::BENEFIT, w, n, 0.0, pot};
    int shift = 0;
    int rc = prepare_parallel(f, pot, pool, &shift);
    if (rc) return rc;
    rc = certified_perfect(f, k, shift, mate_out, pool);
    if (rc) return rc;
    for (int v = 0; v < n; ++v)
        if (mate_out[v] < 0) return -3;
    return 0;
}

}  // extern "C"
