/* Exact Kendall tau pair counts by direct pair enumeration — TEST INFRASTRUCTURE ONLY.
 *
 * C restatement of the reference's O(n^2) row loop (ranksched/ranking.py:45-57):
 * for every pair i < j, s = sign(x_j - x_i) * sign(y_j - y_i); s > 0 concordant,
 * s < 0 discordant; ties within x (n1), within y (n2) and within both (n3) are counted
 * over the same pairs (equal to the np.unique counts for NaN-free input). Rows are
 * dealt round-robin to `threads` pthreads; the counts are sums over rows, so the
 * result does not depend on the split. Used as the checker for the 1M-row golden
 * counts and as bench.py's CPU baseline for tau pairs/s.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    const double* x;
    const double* y;
    int64_t n, t, nt;
    int64_t c, d, n1, n2, n3;
} job_t;

static void* work(void* arg) {
    job_t* j = (job_t*)arg;
    int64_t c = 0, d = 0, n1 = 0, n2 = 0, n3 = 0;
    for (int64_t i = j->t; i < j->n - 1; i += j->nt) {
        const double xi = j->x[i], yi = j->y[i];
        int64_t cc = 0, dd = 0, t1 = 0, t2 = 0, t3 = 0;
        for (int64_t k = i + 1; k < j->n; ++k) {
            const double dx = j->x[k] - xi, dy = j->y[k] - yi;
            const int sx = (dx > 0) - (dx < 0), sy = (dy > 0) - (dy < 0);
            const int p = sx * sy;
            cc += p > 0;
            dd += p < 0;
            t1 += sx == 0;
            t2 += sy == 0;
            t3 += (sx == 0) & (sy == 0);
        }
        c += cc; d += dd; n1 += t1; n2 += t2; n3 += t3;
    }
    j->c = c; j->d = d; j->n1 = n1; j->n2 = n2; j->n3 = n3;
    return 0;
}

/* out = {C, D, n1, n2, n3} */
int tau_pairs_f64(const double* x, const double* y, int64_t n, int64_t* out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (job_t){x, y, n, t, threads, 0, 0, 0, 0, 0};
        if (pthread_create(&th[t], 0, work, &jobs[t])) return -1;
    }
    for (int k = 0; k < 5; ++k) out[k] = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], 0);
        out[0] += jobs[t].c; out[1] += jobs[t].d; out[2] += jobs[t].n1;
        out[3] += jobs[t].n2; out[4] += jobs[t].n3;
    }
    return 0;
}
