/* CPU oracle, compiled -- TEST INFRASTRUCTURE (the checker, never the product).
 *
 * A plain-C restatement of the reference's per-mask stream body for the
 * per-component maximum |W(u, v)|, fast enough to cover EVERY component of
 * the two large BASELINE configs (20x20: 2^20 - 1 masks x 2^20 points;
 * 24x16: 65535 masks x 2^24 points) in minutes on the host cores, where the
 * reference itself needs ~26 core-hours.  Only tests/, __graft_entry__ and
 * bench.py's CPU legs may call it (through oracle/sbw_oracle.py).
 *
 * Reference anchors (/root/reference/pkg/src/sboxeval):
 *   sbox.py:114-116   g_v(x) = popcount(v & S(x)) & 1
 *   sbox.py:145-152   polarity_row: f(x) = 1 - 2 g_v(x)  (int32)
 *   walsh.py:73-104   fwht_column_in_place: natural order, stage j = 1, 2, ..
 *                     (a, b) -> (a + b, a - b) on pairs (i, i + j), (i & j) = 0;
 *                     max |.| over the values of the last stage.  Every
 *                     intermediate of a polarity column is bounded by 2^n <=
 *                     2^24, so int32 arithmetic is exact (no wrap to model).
 *   walsh.py:237-240  the stream loop over v = v_lo .. v_hi - 1
 *
 * Pinned by tests/test_oracle.py: equal to the reference's full 16x16 maxima
 * (65535 components), its sampled 20x20 / 24x16 masks, and every chunk of the
 * reference's own full 20x20 / 24x16 run (tests/golden/full_work/) present.
 *
 * The transform order differs from the reference's (cache blocking: the low
 * B stages inside 2^B-point blocks, then the high stages over column strips);
 * butterfly stages over distinct index bits commute, and with no overflow the
 * result is identical.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef BLK_BITS
#define BLK_BITS 13            /* 32 KiB blocks: stages 0..12 in L1/L2 */
#endif
#ifndef STRIP
#define STRIP 64               /* high stages: 64 int32 (four 64-B lines) per row */
#endif

static inline int32_t iabs32(int32_t x) { return x < 0 ? -x : x; }

/* Stages 0..b-1 of one contiguous block of 2^b points (walsh.py:91-101). */
static void fwht_block(int32_t *a, int b) {
    const int len = 1 << b;
    for (int i = 0; i + 4 <= len; i += 4) { /* stages j = 1, 2 in registers */
        int32_t x0 = a[i], x1 = a[i + 1], x2 = a[i + 2], x3 = a[i + 3];
        int32_t s0 = x0 + x1, d0 = x0 - x1, s1 = x2 + x3, d1 = x2 - x3;
        a[i] = s0 + s1; a[i + 1] = d0 + d1; a[i + 2] = s0 - s1; a[i + 3] = d0 - d1;
    }
    if (len < 4) {
        if (len == 2) { int32_t x0 = a[0], x1 = a[1]; a[0] = x0 + x1; a[1] = x0 - x1; }
        return;
    }
    for (int j = 4; j < len; j <<= 1)
        for (int i = 0; i < len; i += 2 * j) {
            int32_t *lo = a + i, *hi = a + i + j;
            for (int k = 0; k < j; ++k) {
                int32_t x = lo[k], y = hi[k];
                lo[k] = x + y; hi[k] = x - y;
            }
        }
}

/* max |W| of one component: generate f_v, transform, fold (int32 exact). */
static int32_t component_max(const uint32_t *table, int n, uint32_t v, int32_t *buf) {
    const int64_t len = (int64_t)1 << n;
    const int b = n < BLK_BITS ? n : BLK_BITS;
    const int64_t blk = (int64_t)1 << b;
    for (int64_t o = 0; o < len; o += blk) {
        int32_t *a = buf + o;
        for (int64_t x = 0; x < blk; ++x)
            a[x] = 1 - 2 * (int32_t)(__builtin_popcount(table[o + x] & v) & 1);
        fwht_block(a, b);
    }
    int32_t mx = 0;
    if (n <= b) {
        if (len == 1) return iabs32(buf[0]);
        for (int64_t x = 0; x < len; ++x) { int32_t t = iabs32(buf[x]); mx = t > mx ? t : mx; }
        return mx;
    }
    /* High stages b..n-1: for each strip of STRIP consecutive offsets inside a
     * block, the 2^(n-b) rows (one per block) form an independent small WHT. */
    const int hb = n - b;
    const int64_t rows = (int64_t)1 << hb;
    for (int64_t c = 0; c < blk; c += STRIP) {
        int64_t j = 1;
        for (; 4 * j <= rows; j <<= 2)      /* two stages (j, 2j) per sweep */
            for (int64_t r = 0; r < rows; r += 4 * j)
                for (int64_t q = 0; q < j; ++q) {
                    int32_t *p0 = buf + ((r + q) << b) + c, *p1 = buf + ((r + q + j) << b) + c;
                    int32_t *p2 = buf + ((r + q + 2 * j) << b) + c;
                    int32_t *p3 = buf + ((r + q + 3 * j) << b) + c;
                    for (int k = 0; k < STRIP; ++k) {
                        int32_t s0 = p0[k] + p1[k], d0 = p0[k] - p1[k];
                        int32_t s1 = p2[k] + p3[k], d1 = p2[k] - p3[k];
                        p0[k] = s0 + s1; p1[k] = d0 + d1; p2[k] = s0 - s1; p3[k] = d0 - d1;
                    }
                }
        for (; j < rows; j <<= 1)
            for (int64_t r = 0; r < rows; r += 2 * j)
                for (int64_t q = 0; q < j; ++q) {
                    int32_t *lo = buf + ((r + q) << b) + c;
                    int32_t *hi = buf + ((r + q + j) << b) + c;
                    for (int k = 0; k < STRIP; ++k) {
                        int32_t x = lo[k], y = hi[k];
                        lo[k] = x + y; hi[k] = x - y;
                    }
                }
        for (int64_t r = 0; r < rows; ++r) {
            const int32_t *p = buf + (r << b) + c;
            for (int k = 0; k < STRIP; ++k) { int32_t t = iabs32(p[k]); mx = t > mx ? t : mx; }
        }
    }
    return mx;
}

typedef struct {
    const uint32_t *table;
    int n;
    uint32_t v_lo, v_hi;
    int32_t *out;
    volatile uint32_t *next;   /* shared work counter (masks, in chunks) */
    pthread_mutex_t *mu;
    int rc;
} Job;

static void *worker(void *p) {
    Job *j = (Job *)p;
    int32_t *buf = (int32_t *)aligned_alloc(64, (((size_t)4 << j->n) + 63) & ~(size_t)63);
    if (!buf) { j->rc = -1; return NULL; }
    const uint32_t step = j->n >= 20 ? 1 : (j->n >= 16 ? 16 : 256);
    for (;;) {
        pthread_mutex_lock(j->mu);
        uint32_t a = *j->next;
        *j->next = a + step < j->v_hi && a + step > a ? a + step : j->v_hi;
        pthread_mutex_unlock(j->mu);
        if (a >= j->v_hi) break;
        uint32_t b = a + step < j->v_hi && a + step > a ? a + step : j->v_hi;
        for (uint32_t v = a; v < b; ++v) j->out[v - j->v_lo] = component_max(j->table, j->n, v, buf);
    }
    free(buf);
    j->rc = 0;
    return NULL;
}

/* out[v - v_lo] = max_u |W(u, v)| for v in [v_lo, v_hi); table has 2^n
 * entries.  threads <= 0: one.  Returns 0, or -1 on bad arguments / OOM. */
int sbwo_component_max_abs(const uint32_t *table, int n, uint32_t v_lo, uint32_t v_hi,
                           int32_t *out, int threads) {
    if (!table || !out || n < 0 || n > 24 || v_hi < v_lo) return -1;
    if (v_hi == v_lo) return 0;
    if (threads <= 0) threads = 1;
    if ((uint32_t)threads > v_hi - v_lo) threads = (int)(v_hi - v_lo);
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    volatile uint32_t next = v_lo;
    Job *jobs = (Job *)calloc((size_t)threads, sizeof(Job));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int rc = 0;
    for (int i = 0; i < threads; ++i) {
        jobs[i] = (Job){table, n, v_lo, v_hi, out, &next, &mu, 0};
        if (pthread_create(&th[i], NULL, worker, &jobs[i])) { rc = -1; threads = i; break; }
    }
    for (int i = 0; i < threads; ++i) {
        pthread_join(th[i], NULL);
        if (jobs[i].rc) rc = -1;
    }
    free(jobs);
    free(th);
    return rc;
}
