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
// matching) is solved on a SPARSE candidate graph -- the k lightest edges of
// every vertex -- and then certified on the complete graph with the LP dual the
// solver ends with: every edge's reduced cost y_i + y_j + sum of the duals of
// the blossoms containing both ends - w_ij must be >= 0 (the reference's
// verify-optimum condition).  Violating edges are added and the sparse problem
// re-solved, so the result is a certified optimum of the full graph; the work
// is ~n^2 k instead of n^3 (seconds instead of hours at n = 4,096).
#include "cosched_match.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

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

    int run(bool max_cardinality) {
        const int n = n_;
        // initial duals: doubled vertex duals = max weight (the reference init)
        i128 maxw = 0;
        for (const i128 &x : g_.w) maxw = std::max(maxw, x << extra_);
        for (int v = 0; v < n; ++v) dual_[v] = maxw;

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
int choose_shift(const EdgeValue &f, int *shift) {
    int emin = INT32_MAX, emax = INT32_MIN;
    for (int u = 0; u < f.n; ++u)
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
    if (emin == INT32_MAX) { *shift = 0; return 0; }
    const int s = 53 - emin;            // ulp(r) = 2^(e-53) -> integer after << s
    if (emax + s > 96) return -2;       // keep 2^31 of headroom below 2^127 for duals
    *shift = s;
    return 0;
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

int check_square(const double *w, int32_t n) {
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
            const double x = w[(size_t)u * n + v];
            if (!std::isfinite(x)) return -1;
            if (u != v && x != w[(size_t)v * n + u]) return -1;
        }
    return 0;
}

}  // namespace

extern "C" {

const char *cm_version(void) { return "cosched_match 0.3.0 (exact int128 blossom, sparse + dual certificate)"; }

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
    if (check_square(w, n)) return -1;
    double mx = -INFINITY;
    for (size_t q = 0; q < (size_t)n * n; ++q) mx = std::max(mx, w[q]);
    EdgeValue f{EdgeValue::REFLECT, w, n, mx + 1.0, nullptr};   // matcher.py:84
    int shift = 0;
    int rc = choose_shift(f, &shift);
    if (rc) return rc;
    rc = certified_matching(f, k, shift, mate_out);
    if (rc) return rc;
    for (int v = 0; v < n; ++v)
        if (mate_out[v] < 0) return -3;
    return 0;
}

int cm_min_weight_perfect_matching_pot(const double *w, int32_t n, const double *pot, int32_t k,
                                       int32_t *mate_out) {
    if (n < 2 || (n & 1) || !w || !pot || !mate_out) return -1;
    if (check_square(w, n)) return -1;
    for (int u = 0; u < n; ++u) {
        if (!std::isfinite(pot[u])) return -1;
        for (int v = 0; v < n; ++v)
            if (u != v && w[(size_t)u * n + v] > pot[u] + pot[v]) return -4;   // not a potential bound
    }
    EdgeValue f{EdgeValue::BENEFIT, w, n, 0.0, pot};
    int shift = 0;
    int rc = choose_shift(f, &shift);
    if (rc) return rc;
    rc = certified_matching(f, k, shift, mate_out);
    if (rc) return rc;
    // vertices left single pair up in index order: between two of them the
    // benefit is 0, so any pairing completes an optimal perfect matching
    int prev = -1;
    for (int v = 0; v < n; ++v) {
        if (mate_out[v] >= 0) continue;
        if (prev < 0) { prev = v; continue; }
        mate_out[prev] = v;
        mate_out[v] = prev;
        prev = -1;
    }
    return prev < 0 ? 0 : -3;
}

}  // extern "C"
