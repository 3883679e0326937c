/*
 * cosched_match.h -- host C ABI of the native matcher.
 *
 * Replaces the reference's pure-Python Edmonds blossom
 * (matcher._max_weight_matching, matcher.py:180-542) behind
 * matcher.min_weight_perfect_matching (matcher.py:78-88).
 * rank 1: the Python solver is O(n^3) interpreted (63 s at n = 512).
 *
 * The solver is the O(n^3) primal-dual blossom algorithm on a dense complete
 * graph, run in EXACT integer arithmetic: every weight is a finite double,
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

/* The same with an explicit candidate degree: the blossom solver runs on the
 * graph of each vertex's k lightest edges, then its LP dual is checked on ALL
 * n(n-1)/2 edges (reduced cost >= 0, the reference's verify-optimum test);
 * violating edges join the candidate set and the solve repeats, so the result
 * is an optimum of the complete graph.  k <= 0 or k >= n - 1: the complete
 * graph directly.  cm_min_weight_perfect_matching uses k = 24. */
int cm_min_weight_perfect_matching_k(const double *w, int32_t n, int32_t k, int32_t *mate_out);

/* Minimum-weight perfect matching given vertex potentials with
 * w[u][v] <= pot[u] + pot[v] for every pair -- the pair graph of the sweep
 * has them: a pair's weight is min(co-run, solo_u + solo_v), so pot = the
 * per-app solo times.  Every perfect matching pays sum(pot) minus its
 * "benefit" pot[u] + pot[v] - w[u][v] >= 0, so the optimum is a MAXIMUM-weight
 * matching of the benefit graph (only positive edges: pairs that co-run
 * profitably), certified as above, with the leftover vertices paired in index
 * order (zero benefit between them).  This removes the massive degeneracy of
 * time-share pairs (all perfect matchings of them weigh the same), which makes
 * the direct solve slow.  Returns -4 if `pot` is not a bound. */
int cm_min_weight_perfect_matching_pot(const double *w, int32_t n, const double *pot, int32_t k,
                                       int32_t *mate_out);

#ifdef __cplusplus
}
#endif
#endif
