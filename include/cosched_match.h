/*
 * cosched_match.h -- host C ABI of the native matcher.
 *
 * Replaces the reference's pure-Python Edmonds blossom
 * (matcher._max_weight_matching, matcher.py:180-542) behind
 * matcher.min_weight_perfect_matching (matcher.py:78-88).
 * rank 1: the Python solver is O(n^3) interpreted (63 s at n = 512).
 *
 * The solver is the primal-dual blossom algorithm (O(n^3) on a dense graph),
 * run on a sparse candidate graph in EXACT integer arithmetic: every weight is a finite double,
 * scaled by a power of two into a 128-bit integer, so tightness tests are
 * exact and the result is a true optimum of the given doubles.
 */
#ifndef COSCHED_MATCH_H
#define COSCHED_MATCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *cm_version(void);

/* Maximum-weight matching of the complete graph on n vertices with symmetric
 * weights w[i*n + j] (diagonal ignored).  mate_out[v] = partner or -1.
 * Returns 0, or -1 on bad input (non-finite / asymmetric / n < 0),
 * -2 when weights span too many binary orders of magnitude for exact scaling. */
int cm_max_weight_matching(const double *w, int32_t n, int32_t *mate_out);

/* Minimum-weight perfect matching the reference's way (matcher.py:78-88):
 * reflect r = (max(w) + 1) - w over the whole matrix (diagonal included, as
 * numpy does), take the maximum-weight matching of r, which is perfect on a
 * complete graph with an even vertex count.  mate_out as above.
 * Returns 0, -1 on bad input (odd n, n < 2, non-finite, asymmetric), -2 as
 * above, -3 if the matching came out imperfect (internal error). */
int cm_min_weight_perfect_matching(const double *w, int32_t n, int32_t *mate_out);

/* The same with an explicit candidate degree k.  Solved as a maximum-weight
 * PERFECT matching of the reflected values, warm-started and certified:
 *   - an eps-scaling auction on the assignment relaxation (row-parallel host
 *     threads) prices every vertex; from those prices the solver derives
 *     EXACT integer vertex duals feasible on all n(n-1)/2 edges;
 *   - the blossom solver runs on each vertex's k least-slack edges (plus a
 *     backbone that guarantees a perfect matching), starting from those duals
 *     and the tight pairs they imply;
 *   - its LP dual is checked on ALL n(n-1)/2 edges (reduced cost >= 0, the
 *     reference's verify-optimum test); violating edges join the candidate set
 *     and the solve resumes from the previous duals and matching,
 * so the result is an optimum of the complete graph.  k <= 0 or k >= n - 1:
 * the complete graph directly.  cm_min_weight_perfect_matching uses k = 24. */
int cm_min_weight_perfect_matching_k(const double *w, int32_t n, int32_t k, int32_t *mate_out);

/* Minimum-weight perfect matching given vertex potentials with
 * w[u][v] <= pot[u] + pot[v] for every pair -- the pair graph of the sweep
 * has them: a pair's weight is min(co-run, solo_u + solo_v), so pot = the
 * per-app solo times.  Every perfect matching pays sum(pot) minus its
 * "benefit" pot[u] + pot[v] - w[u][v] >= 0, so the optimum is a maximum-weight
 * PERFECT matching of the benefit graph (zero-benefit edges are the pairs that
 * time-share), solved and certified as above.  The benefit form keeps the
 * values small and the auction prices sharp; at n = 4,096 the solve takes
 * ~2 s on 8 host threads.  Returns -4 if `pot` is not a bound. */
int cm_min_weight_perfect_matching_pot(const double *w, int32_t n, const double *pot, int32_t k,
                                       int32_t *mate_out);

#ifdef __cplusplus
}
#endif
#endif
