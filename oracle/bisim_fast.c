/*
 * oracle/bisim_fast.c -- sequential, event-driven restatement of the
 * reference refinement loops, for parity checks at full benchmark size.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as bisim_oracle.c): loaded by tests/
 * and oracle/gen_scale.py, never by the product.
 *
 * The literal oracle (bisim_oracle.c) runs every PRAM phase over all n
 * states / m transitions, as the reference does, so a round costs O(n + m)
 * and configs with 10^5..10^6 rounds take hours.  This file computes the
 * SAME Priority program round by round, but touches only what a round can
 * change:
 *
 *   select   C = smallest unstable label (pram.py:153-154 on bcrp.py:241-242
 *            / rcpp.py:94-95): a binary min-heap over the unstable labels.
 *   mark     mark[slot] := 1 for every in-edge (slot, s) of every member of
 *            block C (bcrp.py:255-258; RCPP: mark[s], rcpp.py:123-127).
 *            Blocks holding a marked state are "touched".
 *   tag      split[s] iff some slot k < nr_marks[s] has mark[off[s]+k] !=
 *            mark[off[leader]+k] (bcrp.py:260-265; RCPP: mark[s] !=
 *            mark[leader], rcpp.py:200).  A block without a marked member
 *            has all marks 0 and cannot split, so only touched blocks are
 *            scanned (every member of them, marked or not).
 *   sub_a/b  unstable[C] := 0; the split members of a block form ONE new
 *            block labelled by its smallest member (Priority), old and new
 *            labels raised, and for BCRP C re-raised if anything split
 *            (bcrp.py:267-283, rcpp.py:196-216).
 *
 * Blocks are kept as contiguous ranges of a member array (split members
 * move to the range's tail), so no phase ever scans all n states.
 * splits_per_iteration[k] = number of blocks that split in round k
 * (bcrp.py:304-306).  The guard counts label rounds + main rounds + the
 * terminal pass exactly like the literal oracle (pram.py:195-200).
 *
 * Pinned in tests/test_oracle_golden.py against the reference fixtures and
 * against the literal oracle on random instances.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_BAD_INPUT = 1, OR_GUARD = 2, OR_NOMEM = 3 };

typedef struct {
    int64_t supersteps;
    int64_t label_rounds;
    int64_t guard_count;
    int32_t initial_blocks;
    int32_t final_blocks;
    int64_t mark_length;
    double t_pre_s;
    double t_label_s;
    double t_loop_s;
} oracle_stats;

/* from bisim_oracle.c */
int64_t oracle_preprocess(int32_t n, int64_t m, int32_t A, const int32_t *src, const int32_t *act,
                          int32_t *perm, int32_t *action_switch, int32_t *order, int32_t *nr_marks,
                          int32_t *off);
int oracle_label_partition(int32_t n, int64_t m, int32_t A, const int32_t *src, const int32_t *act,
                           int32_t *block_out, int threads);

#include <time.h>
static double fnow(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---- min-heap of unstable labels; flag[] dedupes (a label is in the heap
 * iff its flag is set, since only the popped minimum is ever cleared) */
typedef struct {
    int32_t *h;
    int64_t size;
    uint8_t *flag;
} uheap;

static void heap_push(uheap *q, int32_t v) {
    if (q->flag[v]) return;
    q->flag[v] = 1;
    int64_t i = q->size++;
    while (i > 0) {
        int64_t p = (i - 1) >> 1;
        if (q->h[p] <= v) break;
        q->h[i] = q->h[p];
        i = p;
    }
    q->h[i] = v;
}

static int32_t heap_pop(uheap *q) {
    int32_t top = q->h[0];
    q->flag[top] = 0;
    int32_t v = q->h[--q->size];
    int64_t i = 0, sz = q->size;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= sz) break;
        if (c + 1 < sz && q->h[c + 1] < q->h[c]) ++c;
        if (q->h[c] >= v) break;
        q->h[i] = q->h[c];
        i = c;
    }
    if (sz > 0) q->h[i] = v;
    return top;
}

/* ---- blocks as ranges of a member array */
typedef struct {
    int32_t n;
    int32_t *elems; /* states grouped by block */
    int32_t *pos;   /* index of each state in elems */
    int32_t *bstart, *bsize; /* indexed by block label */
    int32_t *block; /* label (leader) of each state */
} parts;

static int parts_init(parts *P, int32_t n, int32_t *block) {
    P->n = n;
    P->block = block;
    P->elems = malloc((size_t)n * 4);
    P->pos = malloc((size_t)n * 4);
    P->bstart = malloc((size_t)n * 4);
    P->bsize = calloc((size_t)n, 4);
    if (!P->elems || !P->pos || !P->bstart || !P->bsize) return OR_NOMEM;
    for (int32_t s = 0; s < n; ++s) P->bsize[block[s]]++;
    int64_t acc = 0;
    for (int32_t b = 0; b < n; ++b) { P->bstart[b] = (int32_t)acc; acc += P->bsize[b]; }
    int32_t *cur = malloc((size_t)n * 4);
    if (!cur) return OR_NOMEM;
    memcpy(cur, P->bstart, (size_t)n * 4);
    for (int32_t s = 0; s < n; ++s) {
        int32_t at = cur[block[s]]++;
        P->elems[at] = s;
        P->pos[s] = at;
    }
    free(cur);
    return OR_OK;
}

static void parts_free(parts *P) {
    free(P->elems); free(P->pos); free(P->bstart); free(P->bsize);
}

/* Move the split members of block b (flagged in split[], listed in
 * splist[0..k)) to the tail of its range as the new block w. */
static void parts_split(parts *P, int32_t b, const int32_t *splist, int32_t k, int32_t w) {
    int32_t end = P->bstart[b] + P->bsize[b];
    for (int32_t i = 0; i < k; ++i) {
        int32_t s = splist[i];
        int32_t dst = end - 1 - i;
        int32_t other = P->elems[dst];
        int32_t ps = P->pos[s];
        P->elems[ps] = other;
        P->pos[other] = ps;
        P->elems[dst] = s;
        P->pos[s] = dst;
        P->block[s] = w;
    }
    P->bsize[b] -= k;
    P->bstart[w] = end - k;
    P->bsize[w] = k;
}

/* One refinement loop for both algorithms.  BCRP: marks live on L slots
 * (slot ranges off[s] .. off[s]+nr[s]); RCPP: one mark per state (off[s]=s,
 * nr[s]=1 for the split test).  rin_ptr/rin_slot/rin_src: in-edges by
 * target, carrying the mark slot and the source. */
static int refine(int32_t n, int bcrp, const int32_t *off, const int32_t *nr,
                  const int32_t *rin_ptr, const int32_t *rin_slot, const int32_t *rin_src,
                  int64_t mark_len, int32_t *block, int64_t max_supersteps, int64_t steps0,
                  int32_t *splits_out, int64_t splits_cap, oracle_stats *st,
                  int64_t nstop, const int64_t *stops, int32_t *blocks_out, uint8_t *unstable_out) {
    int rc = OR_NOMEM;
    parts P;
    memset(&P, 0, sizeof P);
    uheap q = {0};
    uint8_t *mark = calloc((size_t)(mark_len ? mark_len : 1), 1);
    int32_t *marked = malloc((size_t)(mark_len ? mark_len : 1) * 4);
    uint8_t *touched = calloc((size_t)n, 1);
    int32_t *tlist = malloc((size_t)n * 4);
    int32_t *splist = malloc((size_t)n * 4);
    q.h = malloc((size_t)n * 4);
    q.flag = calloc((size_t)n, 1);
    if (!mark || !marked || !touched || !tlist || !splist || !q.h || !q.flag) goto out;
    if (parts_init(&P, n, block) != OR_OK) goto out;
    for (int32_t s = 0; s < n; ++s) heap_push(&q, block[s]); /* leaders (bcrp.py:226-229) */

    int64_t steps = steps0, rounds = 0;
    for (;;) {
        steps += 1; /* begin_superstep */
        if (max_supersteps >= 0 && steps > max_supersteps) {
            rc = OR_GUARD;
            st->guard_count = steps;
            goto out;
        }
        if (q.size == 0) break; /* C = NONE */
        const int32_t C = heap_pop(&q); /* sub_a's unstable[C] := false */
        rounds += 1;
        /* mark */
        int64_t nmarked = 0;
        int32_t ntouched = 0;
        const int32_t cb = P.bstart[C], ce = cb + P.bsize[C];
        for (int32_t i = cb; i < ce; ++i) {
            const int32_t t = P.elems[i];
            for (int32_t e = rin_ptr[t]; e < rin_ptr[t + 1]; ++e) {
                const int32_t slot = rin_slot[e];
                if (mark[slot]) continue;
                mark[slot] = 1;
                marked[nmarked++] = slot;
                const int32_t b = block[rin_src[e]];
                if (!touched[b]) { touched[b] = 1; tlist[ntouched++] = b; }
            }
        }
        /* tag + elect + split, block by block: every touched block's split
         * set depends only on the marks (fixed after the mark phase) and on
         * its own members, so handling blocks one after another equals the
         * phase-synchronous order. */
        int32_t nsplit = 0;
        for (int32_t ti = 0; ti < ntouched; ++ti) {
            const int32_t b = tlist[ti];
            touched[b] = 0;
            const int32_t bb = P.bstart[b], be = bb + P.bsize[b];
            const int32_t lo = off[b], k = nr[b];
            int32_t ns = 0, w = INT32_MAX;
            for (int32_t i = bb; i < be; ++i) {
                const int32_t s = P.elems[i];
                const int32_t so = off[s];
                int differ = 0;
                for (int32_t j = 0; j < k && !differ; ++j) differ = mark[so + j] != mark[lo + j];
                if (differ) {
                    splist[ns++] = s;
                    if (s < w) w = s;
                }
            }
            if (ns == 0) continue;
            nsplit += 1;
            parts_split(&P, b, splist, ns, w);
            heap_push(&q, b); /* unstable[old] */
            heap_push(&q, w); /* unstable[winner] */
        }
        if (bcrp && nsplit > 0) heap_push(&q, C); /* bcrp.py:282 */
        for (int64_t i = 0; i < nmarked; ++i) mark[marked[i]] = 0;
        if (splits_out && rounds <= splits_cap) splits_out[rounds - 1] = nsplit;
        /* checkpoints: the program's state (block, unstable) after round
         * stops[i] -- what the literal oracle resumes from (oracle_set_state) */
        while (nstop > 0 && stops[0] == rounds) {
            memcpy(blocks_out, block, (size_t)n * 4);
            memcpy(unstable_out, q.flag, (size_t)n);
            blocks_out += n;
            unstable_out += n;
            ++stops;
            --nstop;
            if (nstop == 0) goto done;
        }
    }
done:
    st->supersteps = rounds;
    rc = OR_OK;
out:
    parts_free(&P);
    free(mark); free(marked); free(touched); free(tlist); free(splist); free(q.h); free(q.flag);
    return rc;
}

static int32_t nblocks(int32_t n, const int32_t *block) {
    int32_t c = 0;
    for (int32_t s = 0; s < n; ++s) c += block[s] == s;
    return c;
}

/* in-edges by target: (slot, source) */
static int build_rin(int32_t n, int64_t m, const int32_t *esrc, const int32_t *edst,
                     const int32_t *eslot, int32_t **ptr_o, int32_t **slot_o, int32_t **src_o) {
    int32_t *ptr = calloc((size_t)n + 1, 4);
    int32_t *slot = malloc((size_t)(m ? m : 1) * 4);
    int32_t *src = malloc((size_t)(m ? m : 1) * 4);
    if (!ptr || !slot || !src) { free(ptr); free(slot); free(src); return OR_NOMEM; }
    for (int64_t i = 0; i < m; ++i) ptr[edst[i] + 1]++;
    for (int32_t t = 0; t < n; ++t) ptr[t + 1] += ptr[t];
    int32_t *cur = malloc(((size_t)n + 1) * 4);
    if (!cur) { free(ptr); free(slot); free(src); return OR_NOMEM; }
    memcpy(cur, ptr, ((size_t)n + 1) * 4);
    for (int64_t i = 0; i < m; ++i) {
        int32_t at = cur[edst[i]]++;
        slot[at] = eslot[i];
        src[at] = esrc[i];
    }
    free(cur);
    *ptr_o = ptr; *slot_o = slot; *src_o = src;
    return OR_OK;
}

static int bcrp_fast(int32_t n, int64_t m, int32_t A, const int32_t *src, const int32_t *act,
                     const int32_t *dst, int64_t max_supersteps, int32_t *block_out,
                     int32_t *splits_out, int64_t splits_cap, oracle_stats *st, int threads,
                     int64_t nstop, const int64_t *stops, int32_t *blocks_out,
                     uint8_t *unstable_out) {
    memset(st, 0, sizeof(*st));
    if (n < 1 || m < 0 || A < 0) return OR_BAD_INPUT;
    for (int64_t i = 0; i < m; ++i)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n || act[i] < 0 || act[i] >= A)
            return OR_BAD_INPUT;
    if (max_supersteps == INT64_MIN) max_supersteps = 3 * (int64_t)n + A + 8; /* bcrp.py:206-207 */
    int rc = OR_NOMEM;
    const size_t mm = (size_t)(m ? m : 1);
    int32_t *perm = malloc(mm * 4), *sw = malloc(mm * 4), *order = malloc(mm * 4);
    int32_t *nr = malloc((size_t)n * 4), *off = malloc((size_t)n * 4);
    int32_t *eslot = malloc(mm * 4);
    int32_t *rptr = NULL, *rslot = NULL, *rsrc = NULL;
    if (!perm || !sw || !order || !nr || !off || !eslot) goto out;
    double t0 = fnow();
    int64_t L = oracle_preprocess(n, m, A, src, act, perm, sw, order, nr, off);
    if (L < 0) goto out;
    st->mark_length = L;
    /* slot of transition perm[k] = off[src] + order[k] (bcrp.py:219) */
    for (int64_t k = 0; k < m; ++k) eslot[perm[k]] = off[src[perm[k]]] + order[k];
    free(perm); perm = NULL;
    free(sw); sw = NULL;
    free(order); order = NULL;
    if (build_rin(n, m, src, dst, eslot, &rptr, &rslot, &rsrc) != OR_OK) goto out;
    free(eslot); eslot = NULL;
    double t1 = fnow();
    st->t_pre_s = t1 - t0;
    /* pi0: the literal |Act| label rounds (bcrp.py:144-184) */
    st->label_rounds = A;
    if (max_supersteps >= 0 && max_supersteps < A) {
        st->guard_count = max_supersteps + 1;
        rc = OR_GUARD;
        goto out;
    }
    if (A > 0) {
        rc = oracle_label_partition(n, m, A, src, act, block_out, threads);
        if (rc != OR_OK) goto out;
    } else {
        for (int32_t s = 0; s < n; ++s) block_out[s] = 0;
    }
    st->initial_blocks = nblocks(n, block_out);
    double t2 = fnow();
    st->t_label_s = t2 - t1;
    rc = refine(n, 1, off, nr, rptr, rslot, rsrc, L, block_out, max_supersteps, A, splits_out,
                splits_cap, st, nstop, stops, blocks_out, unstable_out);
    st->t_loop_s = fnow() - t2;
    if (rc == OR_OK) st->final_blocks = nblocks(n, block_out);
out:
    free(perm); free(sw); free(order); free(nr); free(off); free(eslot);
    free(rptr); free(rslot); free(rsrc);
    return rc;
}

static int rcpp_fast(int32_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     const int32_t *pi0, int64_t max_supersteps, int32_t *block_out,
                     int32_t *splits_out, int64_t splits_cap, oracle_stats *st,
                     int64_t nstop, const int64_t *stops, int32_t *blocks_out,
                     uint8_t *unstable_out) {
    memset(st, 0, sizeof(*st));
    if (n < 1 || m < 0) return OR_BAD_INPUT;
    for (int64_t i = 0; i < m; ++i)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return OR_BAD_INPUT;
    for (int32_t s = 0; s < n; ++s)
        if (pi0[s] < 0 || pi0[s] >= n || pi0[pi0[s]] != pi0[s]) return OR_BAD_INPUT;
    if (max_supersteps == INT64_MIN) max_supersteps = 3 * (int64_t)n + 9; /* rcpp.py:234-235 */
    int rc = OR_NOMEM;
    int32_t *off = malloc((size_t)n * 4), *nr = malloc((size_t)n * 4);
    int32_t *rptr = NULL, *rslot = NULL, *rsrc = NULL;
    if (!off || !nr) goto out;
    double t0 = fnow();
    for (int32_t s = 0; s < n; ++s) { off[s] = s; nr[s] = 1; } /* one mark per state */
    /* RCPP marks the source itself: slot = source */
    if (build_rin(n, m, src, dst, src, &rptr, &rslot, &rsrc) != OR_OK) goto out;
    for (int32_t s = 0; s < n; ++s) block_out[s] = pi0[s]; /* phase_init: verbatim */
    st->initial_blocks = nblocks(n, block_out);
    st->mark_length = n;
    double t2 = fnow();
    st->t_label_s = t2 - t0;
    rc = refine(n, 0, off, nr, rptr, rslot, rsrc, n, block_out, max_supersteps, 0, splits_out,
                splits_cap, st, nstop, stops, blocks_out, unstable_out);
    st->t_loop_s = fnow() - t2;
    if (rc == OR_OK) st->final_blocks = nblocks(n, block_out);
out:
    free(off); free(nr); free(rptr); free(rslot); free(rsrc);
    return rc;
}

int oracle_bcrp_fast(int32_t n, int64_t m, int32_t A, const int32_t *src, const int32_t *act,
                     const int32_t *dst, int64_t max_supersteps, int32_t *block_out,
                     int32_t *splits_out, int64_t splits_cap, oracle_stats *st, int threads) {
    return bcrp_fast(n, m, A, src, act, dst, max_supersteps, block_out, splits_out, splits_cap, st,
                     threads, 0, NULL, NULL, NULL);
}

int oracle_rcpp_fast(int32_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     const int32_t *pi0, int64_t max_supersteps, int32_t *block_out,
                     int32_t *splits_out, int64_t splits_cap, oracle_stats *st) {
    return rcpp_fast(n, m, src, dst, pi0, max_supersteps, block_out, splits_out, splits_cap, st, 0,
                     NULL, NULL, NULL);
}

/* States (block, unstable flags) of the reference program after rounds
 * stops[0] < stops[1] < ... (nstop of them, each <= the run's length):
 * blocks_out / unstable_out hold nstop * n entries.  bench.py uses them to
 * time the literal oracle on windows from the middle and end of a run. */
int oracle_fast_states(int bcrp, int32_t n, int64_t m, int32_t A, const int32_t *src,
                       const int32_t *act, const int32_t *dst, const int32_t *pi0, int64_t nstop,
                       const int64_t *stops, int32_t *blocks_out, uint8_t *unstable_out,
                       int threads) {
    oracle_stats st;
    int32_t *block = malloc((size_t)n * 4);
    if (!block) return OR_NOMEM;
    int rc = bcrp ? bcrp_fast(n, m, A, src, act, dst, -1, block, NULL, 0, &st, threads, nstop,
                              stops, blocks_out, unstable_out)
                  : rcpp_fast(n, m, src, dst, pi0, -1, block, NULL, 0, &st, nstop, stops,
                              blocks_out, unstable_out);
    free(block);
    return rc;
}
