/*
 * bisim.h -- C ABI of libbisim.so, the B200 (sm_100a) implementation of the
 * CRCW-PRAM partition-refinement path of arXiv 2105.11788.
 *
 * Drop-in boundary.  The reference `parbisim` exposes this path as two
 * Python functions:
 *
 *   bcrp_run(lts, policy, *, common_election, observer, max_supersteps)
 *       /root/reference/pkg/src/parbisim/bcrp.py:192-195
 *   rcpp_run(rel, policy, *, common_election, observer, max_supersteps)
 *       /root/reference/pkg/src/parbisim/rcpp.py:220-223
 *
 * both returning (Partition, RunStats) (lts.py:76-114, lts.py:164-184).  The
 * functions below replace the bodies of those two calls: transition arrays
 * in, per-state leader block ids plus the RunStats fields out.  Arrays are
 * plain C-contiguous int32; no torch or CUDA types appear in the signatures.
 *
 * Semantics (bit-exact with the reference under the Priority write policy,
 * pram.py:153-154, which Common-with-election reproduces identically):
 *   - block_out[s] is the leader (minimum state, for canonical inputs) of
 *     s's block; BCRP output is canonical, RCPP keeps pi0's leaders.
 *   - st->supersteps counts main-loop rounds that selected a splitter;
 *     splits_out[k] is the number of blocks split in round k+1.
 *   - The superstep guard counts like PramEngine.begin_superstep
 *     (pram.py:195-200): BCRP completes iff |Act| + R + 1 <= max_supersteps
 *     (default 3n + |Act| + 8, bcrp.py:206-207); RCPP iff R + 1 <=
 *     max_supersteps (default 3n + 9, rcpp.py:234-235).
 *
 * Return codes map to the reference's exceptions: BISIM_BAD_INPUT ->
 * ValueError (lts.py:40-52, rcpp.py:49-55), BISIM_GUARD ->
 * SuperstepLimitError (pram.py:70-71), BISIM_CUDA -> RuntimeError,
 * BISIM_ABORTED -> the observer's own exception.  bisim_last_error()
 * returns a thread-local message for the last failing call.
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns BISIM_CUDA.
 */
#ifndef BISIM_H
#define BISIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BISIM_OK 0
#define BISIM_BAD_INPUT 1
#define BISIM_GUARD 2
#define BISIM_CUDA 3
#define BISIM_ABORTED 4

/* max_supersteps value meaning "the reference default" (max_supersteps=None) */
#define BISIM_DEFAULT_GUARD INT64_MIN

/* Execution strategies of the refinement loop. */
#define BISIM_MODE_AUTO 0
#define BISIM_MODE_PERSISTENT 1 /* one cooperative kernel runs every round (work-efficient) */
#define BISIM_MODE_STEPPED 2    /* one launch per round (observer support) */
#define BISIM_MODE_DENSE 3      /* persistent, every round scans all n states */

typedef struct bisim_stats {
    int64_t supersteps;      /* RunStats.supersteps */
    int64_t label_rounds;    /* |Act| label pre-partition rounds (BCRP) */
    int64_t guard_count;     /* superstep counter when BISIM_GUARD fired */
    int32_t initial_blocks;  /* RunStats.initial_block_count */
    int32_t final_blocks;    /* RunStats.final_block_count */
    int64_t mark_length;     /* BcrpAux.mark_length (n for RCPP) */
    double t_h2d_ms;         /* CUDA-event times on the library stream */
    double t_pre_ms;
    double t_label_ms;
    double t_alg_ms;
    double t_d2h_ms;
    int64_t bytes_alg;       /* algorithmic bytes of the main loop */
    int32_t kernel_launches; /* kernels this call launched */
    int32_t mode;            /* BISIM_MODE_* actually used */
    int64_t rounds_retired;  /* no-op rounds retired in bulk (counted in supersteps) */
} bisim_stats;

/* observer(iteration, block, n, user): called after every counted round in
 * stepped mode with a host copy of the block array (bcrp.py:307-308).  A
 * non-zero return aborts the run with BISIM_ABORTED. */
typedef int (*bisim_observer_fn)(int64_t iteration, const int32_t *block, int32_t n, void *user);

/* Loop-variant flags (bisim_options.flags).  None changes a result: each
 * selects another schedule of the same Priority program, and the parity
 * tests run every variant against the oracle. */
#define BISIM_FLAG_NO_SKIP 1u              /* run no-op rounds one by one (no bulk retirement) */
#define BISIM_FLAG_NO_SOLO 2u              /* every round on the whole grid (no CTA-solo stretches) */
#define BISIM_FLAG_CTA_MAJOR 4u            /* phase-B work items CTA-major */
#define BISIM_FLAG_LITERAL_LABEL_ROUNDS 8u /* label pre-partition as |Act| literal rounds */
#define BISIM_FLAG_WIDE_LAYOUT 16u         /* phase B: 128-member chunks even for small touched blocks */
#define BISIM_FLAG_TWO_PASS 32u            /* phase B: the two-pass (tag, grid barrier, compact) split */
#define BISIM_FLAG_BATCH_WALK 64u          /* phase A: batch registration wave for every grid splitter */

typedef struct bisim_options {
    int32_t device;          /* CUDA ordinal */
    int32_t mode;            /* BISIM_MODE_* */
    bisim_observer_fn observer;
    void *observer_user;
    uint32_t flags;          /* BISIM_FLAG_* (0 = default schedule) */
    int32_t reserved;
} bisim_options;

/* ---- host-pointer entry points (the reference-facing boundary) ---------- */

/* bcrp_run: transitions (src[i], act[i], dst[i]), i < m, act in [0, num_actions). */
int bisim_bcrp(int32_t n, int64_t m, int32_t num_actions, const int32_t *src, const int32_t *act,
               const int32_t *dst, int64_t max_supersteps, int32_t *block_out,
               int32_t *splits_out, int64_t splits_cap, bisim_stats *st, int device);

/* rcpp_run: edges (src[i], dst[i]) and pi0 in leader form (rcpp.py:38-55). */
int bisim_rcpp(int32_t n, int64_t m, const int32_t *src, const int32_t *dst,
               const int32_t *pi0_leader, int64_t max_supersteps, int32_t *block_out,
               int32_t *splits_out, int64_t splits_cap, bisim_stats *st, int device);

/* Same, with options (observer / forced mode). opt may be NULL. */
int bisim_bcrp_ex(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                  const int32_t *act, const int32_t *dst, int64_t max_supersteps,
                  int32_t *block_out, int32_t *splits_out, int64_t splits_cap, bisim_stats *st,
                  const bisim_options *opt);
int bisim_rcpp_ex(int32_t n, int64_t m, const int32_t *src, const int32_t *dst,
                  const int32_t *pi0_leader, int64_t max_supersteps, int32_t *block_out,
                  int32_t *splits_out, int64_t splits_cap, bisim_stats *st,
                  const bisim_options *opt);

/* ---- device-pointer entry points (inputs already resident in HBM) ------- */
/* src/act/dst/pi0 and block_out are device pointers on opt->device;
 * splits_out is a host pointer.  The call is synchronous. */
int bisim_bcrp_device(int32_t n, int64_t m, int32_t num_actions, const int32_t *d_src,
                      const int32_t *d_act, const int32_t *d_dst, int64_t max_supersteps,
                      int32_t *d_block_out, int32_t *splits_out, int64_t splits_cap,
                      bisim_stats *st, const bisim_options *opt);
int bisim_rcpp_device(int32_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst,
                      const int32_t *d_pi0_leader, int64_t max_supersteps, int32_t *d_block_out,
                      int32_t *splits_out, int64_t splits_cap, bisim_stats *st,
                      const bisim_options *opt);

/* ---- transition-sharded mode ----------------------------- */
/* One LTS refined by nshards replicas on devices[0..nshards) (1..8; a
 * device may repeat, which runs several replicas on one GPU for testing).
 * Every replica keeps the whole partition state; the in-edges are split by
 * source range (about m / nshards each) and every round's marks are OR-ed
 * into all replicas over peer memory inside the persistent kernels, with one
 * cross-replica barrier per round.  Same results and RunStats as bisim_bcrp /
 * bisim_rcpp (host pointers; no observer).  flags: BISIM_SHARD_VERIFY also
 * checks that every replica ends with the same partition. */
#define BISIM_SHARD_VERIFY 1
int bisim_bcrp_sharded(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                       const int32_t *act, const int32_t *dst, int64_t max_supersteps,
                       int32_t *block_out, int32_t *splits_out, int64_t splits_cap,
                       bisim_stats *st, const int32_t *devices, int32_t nshards, int32_t flags);
int bisim_rcpp_sharded(int32_t n, int64_t m, const int32_t *src, const int32_t *dst,
                       const int32_t *pi0_leader, int64_t max_supersteps, int32_t *block_out,
                       int32_t *splits_out, int64_t splits_cap, bisim_stats *st,
                       const int32_t *devices, int32_t nshards, int32_t flags);

/* ---- preprocessing tables (bcrp.py:116-126, BcrpAux) -------------------- */
/* Per ORIGINAL transition index i: order_out[i] = rank of act[i] among
 * src[i]'s distinct labels; per state: nr_marks_out[s], off_out[s].  Returns
 * BISIM_OK and *mark_length.  Host pointers. */
int bisim_preprocess(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                     const int32_t *act, int32_t *order_out, int32_t *nr_marks_out,
                     int32_t *off_out, int64_t *mark_length, int device);

/* preprocess(lts) -> BcrpAux in the reference's layout (bcrp.py:116-126):
 * the transitions stably sorted by (source, action) (bcrp.py:49-52; GPU
 * radix sort), perm_out[k] = original index of sorted transition k, the
 * sorted columns, action_switch_out[k] (bcrp.py:55-65) and order_out[k]
 * (bcrp.py:91-104) per SORTED transition, nr_marks_out[s] and off_out[s]
 * (exclusive scan, bcrp.py:105-112) per state, *mark_length = L.  Any
 * output pointer may be NULL.  Host pointers. */
int bisim_preprocess_sorted(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                            const int32_t *act, const int32_t *dst, int32_t *perm_out,
                            int32_t *src_out, int32_t *act_out, int32_t *dst_out,
                            int32_t *action_switch_out, int32_t *order_out,
                            int32_t *nr_marks_out, int32_t *off_out, int64_t *mark_length,
                            int device);

/* partition_by_outgoing_labels(lts, Priority) (bcrp.py:129-141): only the
 * label kernels run (validation, label sets, canonical grouping). */
int bisim_label_partition(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                          const int32_t *act, int32_t *block_out, int device);

/* The label pre-partition under the plain Common policy (bcrp.py:144-184
 * with common_election=False; pram.py:147-152): the literal |Act| rounds,
 * stopped at the first round whose elect phase has two states of one block
 * writing different new leaders.  On a conflict: *conflict_round = that
 * round (0-based), *conflict_leader = the block's leader (the reference's
 * address ("new_leader", leader) -- the conflicting block whose smallest
 * disagreeing state is smallest), *conflict_winner = that smallest state,
 * and block_out = the partition after the round (the conflicting values
 * are the states with block_out == *conflict_winner).  Without a conflict
 * *conflict_round = -1 and block_out = the label partition. */
int bisim_label_rounds_common(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                              const int32_t *act, int32_t *conflict_round, int32_t *conflict_leader,
                              int32_t *conflict_winner, int32_t *block_out, int device);

/* ---- the steps either side of the path ------------------ */
/* quotient(lts, partition) (aut.py:132-152): one state per block, blocks
 * numbered densely in increasing leader order, duplicate (block, action,
 * block) transitions merged keeping first occurrences in transition order.
 * block is a leader-form partition (lts.py:88-94, else BISIM_BAD_INPUT).
 * q_src/q_act/q_dst hold at least m entries; *q_m <= m transitions are
 * written.  Host pointers. */
int bisim_quotient(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                   const int32_t *act, const int32_t *dst, const int32_t *block,
                   int32_t initial_state, int32_t *q_n, int64_t *q_m, int32_t *q_src,
                   int32_t *q_act, int32_t *q_dst, int32_t *q_initial, int device);

/* is_stable(lts, partition) (oracle.py:128-141): *stable_out = 1 iff every
 * state sees the same set of (action, target block) pairs as its leader. */
int bisim_is_stable(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                    const int32_t *act, const int32_t *dst, const int32_t *block,
                    int32_t *stable_out, int device);

/* is_stable_under(lts, partition, states) (oracle.py:144-154): *stable_out = 1
 * iff every state reaches the set `states` (num_states ids; ids outside
 * 0..n-1 are never reached) via the same actions as its leader. */
int bisim_is_stable_under(int32_t n, int64_t m, int32_t num_actions, const int32_t *src,
                          const int32_t *act, const int32_t *dst, const int32_t *block,
                          const int32_t *states, int64_t num_states, int32_t *stable_out,
                          int device);

/* partition_from_assignment(assignment) (lts.py:117-128): states sharing an
 * id share a block, whose leader is its smallest state. */
int bisim_canonical(int32_t n, const int64_t *assignment, int32_t *block_out, int device);

/* ---- .aut ingestion (aut.py:79-92) ---------------- */
/* parse_aut(text): header "des (<initial>, <m>, <n>)" then m lines
 * "(<source>, <label>, <target>)"; action ids follow the sorted label
 * strings (lts.py:69-70).  Multi-threaded host C++ (threads <= 0: all
 * cores).  On a malformed input returns BISIM_BAD_INPUT, bisim_last_error()
 * holds the reference's ParseError message without its "line N: " prefix
 * and info->error_line holds N (0 when the error has no line). */
typedef struct bisim_aut bisim_aut;
typedef struct bisim_aut_info {
    int32_t n;
    int32_t initial_state;
    int64_t m;
    int32_t num_actions;
    int32_t pad;
    int64_t error_line;
} bisim_aut_info;
int bisim_aut_parse(const char *text, int64_t len, int32_t threads, bisim_aut **out,
                    bisim_aut_info *info);
/* Same, reading (mmap) a file. */
int bisim_aut_read_file(const char *path, int32_t threads, bisim_aut **out, bisim_aut_info *info);
/* Copies the m transitions into caller arrays of info->m entries. */
int bisim_aut_columns(const bisim_aut *aut, int32_t *src, int32_t *act, int32_t *dst);
/* Label of action id `action` (UTF-8, *len bytes, not NUL-terminated). */
const char *bisim_aut_label(const bisim_aut *aut, int32_t action, int64_t *len);
void bisim_aut_free(bisim_aut *aut);

/* ---- misc ---------------------------------------------------------------- */
const char *bisim_last_error(void);
int bisim_device_count(void);
/* The library's CUDA stream on `device` (a cudaStream_t), so callers can
 * bracket calls with their own CUDA events.  NULL on error. */
void *bisim_stream(int device);
/* Library version string (build id). */
const char *bisim_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BISIM_H */
