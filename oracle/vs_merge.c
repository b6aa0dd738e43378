/*
 * oracle/vs_merge.c -- TEST INFRASTRUCTURE ONLY (CPU checker, never shipped).
 *
 * Plain-C restatement of the reference's Vertical-Slash point-range merge
 * (Alg. 4), /root/reference/pkg/src/sparseprefill/vs_index.py:28-95:
 *
 *   for each query-block row r (q_start = r*B, q_end = min(q_start+B, S)):
 *     walk slash offsets (descending) -> ranges [max(0,q_start-o), q_end-o),
 *       skipping o >= q_end (vs_index.py:71-72);
 *     coalesce when rs <= cur_end or rs < cover_end(cur) (vs_index.py:78);
 *     flush(cs, ce): points < cover_end are consumed (those < cs become
 *       residual columns, the rest are absorbed, vs_index.py:58-63), then
 *       tiles cs, cs+B, ... while s < ce (vs_index.py:64-68);
 *     trailing points < q_end become columns (vs_index.py:85-90).
 *
 * Used by tests (as the bit-exact checker for the CUDA merge at sizes where
 * the pure-Python restatement is too slow) and by bench.py's CPU legs.
 *
 * Two-phase API (count, then fill) so callers can size the CSR exactly.
 */
#include <stdint.h>

static int64_t cover_end_of(int64_t cs, int64_t ce, int64_t b) {
    return cs + ((ce - cs + b - 1) / b) * b;
}

/* Process one row; when tiles/cols are NULL only counts are produced.
 * Returns the merge-loop op count (vs_index.py ops_per_row). */
static int64_t merge_row(const int64_t *pts, int64_t np, const int64_t *sl, int64_t ns,
                         int64_t r, int64_t S, int64_t b,
                         int64_t *tiles, int64_t *nt, int64_t *cols, int64_t *nc) {
    int64_t q_start = r * b;
    int64_t q_end = q_start + b < S ? q_start + b : S;
    int64_t jv = 0, ops = 0, t = 0, c = 0;
    int have = 0;
    int64_t cur_s = 0, cur_e = 0;
    for (int64_t i = 0; i <= ns; ++i) {
        int64_t rs = 0, re = 0;
        int flush_now = 0, last = (i == ns);
        if (!last) {
            int64_t o = sl[i];
            if (o >= q_end) continue;
            ops++;
            rs = q_start - o > 0 ? q_start - o : 0;
            re = q_end - o;
            if (!have) { cur_s = rs; cur_e = re; have = 1; continue; }
            if (rs <= cur_e || rs < cover_end_of(cur_s, cur_e, b)) {
                if (re > cur_e) cur_e = re;
                continue;
            }
            flush_now = 1;
        } else {
            if (!have) break;
            flush_now = 1;
        }
        if (flush_now) {
            int64_t cov = cover_end_of(cur_s, cur_e, b);
            while (jv < np && pts[jv] < cov) {
                if (pts[jv] < cur_s) { if (cols) cols[c] = pts[jv]; c++; }
                jv++; ops++;
            }
            for (int64_t s = cur_s; s < cur_e; s += b) { if (tiles) tiles[t] = s; t++; ops++; }
            if (!last) { cur_s = rs; cur_e = re; }
        }
    }
    while (jv < np) {
        if (pts[jv] < q_end) { if (cols) cols[c] = pts[jv]; c++; }
        jv++; ops++;
    }
    *nt = t; *nc = c;
    return ops;
}

/* Counts per row: tile_counts[n_rows], col_counts[n_rows], ops[n_rows] (ops may be NULL). */
void oracle_vs_count(const int64_t *pts, int64_t np, const int64_t *sl, int64_t ns,
                     int64_t S, int64_t b, int64_t *tile_counts, int64_t *col_counts,
                     int64_t *ops) {
    int64_t n_rows = (S + b - 1) / b;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t nt, nc;
        int64_t o = merge_row(pts, np, sl, ns, r, S, b, 0, &nt, 0, &nc);
        tile_counts[r] = nt; col_counts[r] = nc;
        if (ops) ops[r] = o;
    }
}

/* Fill CSR given exclusive offsets (length n_rows+1). */
void oracle_vs_fill(const int64_t *pts, int64_t np, const int64_t *sl, int64_t ns,
                    int64_t S, int64_t b, const int64_t *tile_off, const int64_t *col_off,
                    int64_t *tiles, int64_t *cols) {
    int64_t n_rows = (S + b - 1) / b;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t nt, nc;
        merge_row(pts, np, sl, ns, r, S, b, tiles + tile_off[r], &nt, cols + col_off[r], &nc);
    }
}
