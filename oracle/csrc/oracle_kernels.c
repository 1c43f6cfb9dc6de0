/* Oracle C helpers -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain sequential C restatements of the two pure-Python loops of the
 * reference whose run time would otherwise make the oracle impractical at
 * the BASELINE sizes:
 *   o_ilu0       reference linalg.py:178-222  (IKJ ILU(0) on the stored pattern)
 *   o_aggregate  reference linalg.py:279-324  (strength graph + 3-pass greedy aggregation)
 * Compiled with -ffp-contract=off so every `a -= l*u` is a separate multiply
 * and subtract, exactly like the Python float arithmetic it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

/* returns 0 ok, 1 missing diagonal (row in *bad), 2 zero pivot (row in *bad) */
int o_ilu0(int n, const int32_t *indptr, const int32_t *indices, double *data, int64_t *bad)
{
    int64_t *diag = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int rc = 0;
    for (int i = 0; i < n; ++i) {
        diag[i] = -1;
        pos[i] = -1;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
            if (indices[p] == i) diag[i] = p;
        if (diag[i] < 0) { *bad = i; rc = 1; goto done; }
    }
    for (int i = 0; i < n; ++i) {
        const int64_t s = indptr[i], e = indptr[i + 1];
        for (int64_t p = s; p < e; ++p) pos[indices[p]] = p;
        for (int64_t p = s; p < e; ++p) {
            const int k = indices[p];
            if (k >= i) break;
            const double piv = data[diag[k]];
            if (piv == 0.0) { *bad = k; rc = 2; goto done; }
            const double l = data[p] / piv;
            data[p] = l;
            for (int64_t q = diag[k] + 1; q < indptr[k + 1]; ++q) {
                const int64_t t = pos[indices[q]];
                if (t >= 0) data[t] -= l * data[q];
            }
        }
        for (int64_t p = s; p < e; ++p) pos[indices[p]] = -1;
        if (data[diag[i]] == 0.0) { *bad = i; rc = 2; goto done; }
    }
done:
    free(diag);
    free(pos);
    return rc;
}

/* aggregate ids into agg[n]; returns number of aggregates */
int64_t o_aggregate(int n, const int32_t *indptr, const int32_t *indices, const double *data,
                    double theta, int64_t *agg)
{
    int64_t nnz = indptr[n];
    int32_t *nb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    int64_t *nbp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t w = 0;
    nbp[0] = 0;
    for (int i = 0; i < n; ++i) {
        double mx = 0.0;
        int any = 0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            if (indices[p] == i) continue;
            double v = fabs(data[p]);
            if (!any || v > mx) mx = v;
            any = 1;
        }
        if (any) {
            const double thr = theta * mx;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                if (indices[p] == i) continue;
                if (fabs(data[p]) >= thr) nb[w++] = indices[p];
            }
        }
        nbp[i + 1] = w;
    }
    for (int i = 0; i < n; ++i) agg[i] = -1;
    int64_t next = 0;
    for (int i = 0; i < n; ++i) {           /* pass 1: seeds with free neighbourhoods */
        if (agg[i] != -1) continue;
        int free_nb = 1;
        for (int64_t p = nbp[i]; p < nbp[i + 1]; ++p)
            if (agg[nb[p]] != -1) { free_nb = 0; break; }
        if (!free_nb) continue;
        agg[i] = next;
        for (int64_t p = nbp[i]; p < nbp[i + 1]; ++p) agg[nb[p]] = next;
        ++next;
    }
    for (int i = 0; i < n; ++i) {           /* pass 2: first aggregated strong neighbour */
        if (agg[i] != -1) continue;
        for (int64_t p = nbp[i]; p < nbp[i + 1]; ++p)
            if (agg[nb[p]] != -1) { agg[i] = agg[nb[p]]; break; }
    }
    for (int i = 0; i < n; ++i)             /* pass 3: singletons */
        if (agg[i] == -1) agg[i] = next++;
    free(nb);
    free(nbp);
    return next;
}
