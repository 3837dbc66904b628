/*
 * ltl_core.h -- C ABI of the B200 screening core (libltlcore.so).
 *
 * This is the drop-in boundary for the hot path of the reference learner: the object returned by
 *   ltllearn.kernels.make_core(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k,
 *                              budget_bytes, backend)                       (reference kernels.py:140-172)
 * whose contract is spelled out by the reference's two interchangeable cores,
 *   ltllearn._speedups.Core   (reference _speedups.pyx:61-380, Cython/C++)  and
 *   ltllearn._kernels_py.PyCore (reference _kernels_py.py:32-281).
 * Every entry point below names the reference member it replaces.  Paths are relative to
 * /root/reference/pkg/src/ltllearn/.
 *
 * Conventions
 *   - plain C types only; all buffers are HOST pointers owned by the caller; the core copies in / out.
 *   - a characteristic matrix (CM) is uint64[R*W], row-major (word w of row r at cm[r*W + w]); trace
 *     position j of a row lives in word j/64 at bit 63 - j%64.  W == 1 is exactly the reference's uint64[R].
 *   - every function returns LTL_OK (0) or a negative LTL_ERR_* code; the message for the last failure
 *     on a handle is available from ltl_core_last_error().  No exception crosses the ABI.
 *   - a handle is single-threaded and not re-entrant (like the reference core, which holds the GIL).
 *   - the library talks to the GPU only; there is no CPU fallback.  Without a usable CUDA device
 *     ltl_core_create() fails with LTL_ERR_CUDA.
 */
#ifndef LTL_CORE_H
#define LTL_CORE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTL_ABI_VERSION 1

#if defined(__GNUC__)
#define LTL_API __attribute__((visibility("default")))
#else
#define LTL_API
#endif

/* status codes of the screening calls: reference kernels.py:43-45 */
#define LTL_S_DONE 0
#define LTL_S_SOLVED 1
#define LTL_S_OOM 2
/* not in the reference's status set: a deadline armed with the "deadline_ms" option passed between two passes of a cost
 * level -- where the reference raises TimeoutExceeded between its chunks (enumerator.py:154-156, 278, 290).  What earlier
 * passes admitted stays admitted; the caller abandons the search. */
#define LTL_S_TIMEOUT 3

/* fingerprint variants: reference kernels.py:39-41 */
#define LTL_V_GATHER 0
#define LTL_V_MUELLER 1
#define LTL_V_FKP 2
/* not in the reference: this build's NH hash for matrices of more than 64 words, where the reference defines
 * nothing (it refuses such inputs, enumerator.py:70-73).  Definition: oracle/ltl_oracle.c fp_nh, DESIGN.md 3. */
#define LTL_V_NH 3
/* NH over row pairs, for specifications whose traces all have at most 32 positions (one word per row, W == 1):
 * the core then stores two rows per 64-bit word (uint32 storage for L <= 32) and moves half the bytes per matrix.
 * The ABI is unchanged -- matrices cross it as uint64[R].  Definition: oracle/ltl_oracle.c fp_nh32. */
#define LTL_V_NH32 4

/* error codes */
#define LTL_OK 0
#define LTL_ERR_ARG (-1)        /* bad argument (the reference raises ValueError / IndexError) */
#define LTL_ERR_CUDA (-2)       /* CUDA runtime / driver failure, no device */
#define LTL_ERR_BUDGET (-3)     /* add_entry over the logical budget (the reference raises CoreOOM, _speedups.pyx:275-276) */
#define LTL_ERR_DEVICE_OOM (-4) /* device memory exhausted before the logical budget */
#define LTL_ERR_INVARIANT (-5)  /* debug builds of the data: a stored matrix has bits outside the validity masks -- the reference's
                                 * LTLLEARN_DEBUG_MASKS assertion (bitsem.py:46-61); checked when that variable is set in the
                                 * environment or after ltl_core_set_option(h, "debug_masks", 1) */

typedef struct ltl_core ltl_core;

/* One run of candidates of a cost level, in enumeration order (reference enumerator.py:271-296 dispatches
 * exactly these to screen_unary / screen_binary, chunked):  op applied to left entries [a0, a1) and, for
 * binary ops, right entries [b0, b1); b0 = b1 = -1 for unary ops; tri != 0 restricts to right index >
 * left index (reference _speedups.pyx:367). */
typedef struct ltl_segment {
    int32_t op;
    int32_t tri;
    int64_t a0, a1;
    int64_t b0, b1;
} ltl_segment;

/* kernel classes for ltl_core_kernel_stats */
#define LTL_K_SCREEN 0      /* evaluate + check + fingerprint + file in the uniqueness table ("phase A") */
#define LTL_K_FINALIZE 1    /* row-split runs only: combine partial fingerprints */
#define LTL_K_RESOLVE 2     /* which candidate owns its fingerprint */
#define LTL_K_SCAN 3        /* ordered compaction offsets */
#define LTL_K_EMIT 4        /* records of the winners */
#define LTL_K_MATERIALIZE 5 /* append the winners' matrices ("phase B") */
#define LTL_K_REHASH 6
#define LTL_K_PURGE 7
#define LTL_K_MISC 8        /* import / export / record fix-ups */
#define LTL_K_LEVELS 9      /* the first (small) cost levels of a search in one launch: plan + screen + admit + append */
#define LTL_K_COUNT 10

LTL_API int ltl_abi_version(void);

/* Number of CUDA devices visible, or a negative LTL_ERR_* code. */
LTL_API int ltl_device_count(void);

/* Trace packing on the device -- replaces TraceContext.from_traces (reference bitsem.py:73-88; length masks
 * bitsem.py:51-55), generalised to W words per row (position j -> word j/64, bit 63 - j%64).
 * chars: R rows of L characters (uint16 proposition bitmasks, row-major; entries at positions >= lengths[r] are
 * ignored), lengths: R trace lengths.  Writes masks_out[R*W] and atoms_out[n_props][R*W] (host buffers).
 * 1 <= n_props <= 16, L <= 64*W.  No core handle is involved; errors via ltl_core_last_error(NULL). */
LTL_API int ltl_pack_traces(const uint16_t* chars, const int64_t* lengths, int64_t R, int L, int n_props, int W, int device,
                            uint64_t* masks_out, uint64_t* atoms_out);

/* ---- Device-resident specification (for specifications of many traces; no reference counterpart as an object) -------
 * What the reference does on the host before a search, done on the device so that a 2^21-trace specification is
 * uploaded once and nothing comes back but counters:
 *   ltl_traces_create  uploads the character matrices (positives, then negatives: the row order of every matrix,
 *                      reference traces.py:81-83; both uint16[rows][L], entries at positions >= length ignored), hashes
 *                      every trace to 128 bits and files the hashes with atomicMin(row): rows that are not the first
 *                      holder of their hash are SUSPECTS of being duplicates (reference traces.py:64-106 de-duplicates
 *                      per side and refuses P and N sharing a trace) -- the host compares exactly those few rows;
 *                      also the census of the closed-form overfit cost (reference formula.py:230-250)
 *   ltl_traces_pack    trace packing (reference bitsem.py:73-88) into device-resident masks / atoms, plus the error
 *                      counts of every bare proposition and its negation (atom fast path, enumerator.py:182-192)
 *   ltl_traces_info    out[48]: 0 rows, 1 positives, 2 words per row, 3 max length, 4 min length, 5 non-empty traces,
 *                      6 OR of all characters, 7 positions of the positive traces, 8 set proposition bits of the positive
 *                      traces, 9 suspects, 10 empty positive traces, 11 propositions packed, 12 / 13 bytes copied
 *                      host->device / device->host, 16 + p errors of proposition p, 32 + p errors of its negation
 *   ltl_traces_suspects  (row, first row with the same hash) pairs, returns how many were written
 *   ltl_traces_export  host copies of the packed masks[R*W] and atoms[n_props][R*W] (tools, tests)
 *   ltl_core_create_on_traces / ltl_core_add_atom  a core over the packed traces (masks stay in HBM) and the
 *                      admission of a proposition's matrix (negated != 0: its negation inside the mask, for the NNF
 *                      fragment, reference enumerator.py:223-230) -- add_entry without the host round trip */
typedef struct ltl_traces ltl_traces;
LTL_API int ltl_traces_create(const uint16_t* pos_chars, const int64_t* pos_lengths, int64_t n_pos, const uint16_t* neg_chars,
                              const int64_t* neg_lengths, int64_t n_neg, int L, int device, ltl_traces** out);
LTL_API void ltl_traces_destroy(ltl_traces* t);
LTL_API const char* ltl_traces_last_error(const ltl_traces* t); /* t may be NULL: last create() failure */
LTL_API int ltl_traces_pack(ltl_traces* t, int n_props);
LTL_API int ltl_traces_info(ltl_traces* t, uint64_t out[48]);
LTL_API int ltl_traces_suspects(ltl_traces* t, int64_t* pairs, int64_t cap_pairs);
LTL_API int ltl_traces_export(ltl_traces* t, uint64_t* masks_out, uint64_t* atoms_out);
LTL_API int ltl_core_create_on_traces(ltl_traces* t, int err_max, int variant, const int32_t* proj_rows,
                                      const int32_t* proj_offs, int n_proj, int fkp_bits, int mask_k, uint64_t budget_bytes,
                                      ltl_core** out);
LTL_API int ltl_core_add_atom(ltl_core* h, ltl_traces* t, int prop, int negated, int op, int lhs, int rhs, int64_t* index_out);

/* Trace files (reference traces.py:180-253: one trace per line, positions separated by ';', each position a
 * comma-separated 0/1 vector over the alphabet, a '---' line between positives and negatives; later sections ignored).
 * Host code, two passes over the file's bytes: scan sizes the matrices (traces per side, longest trace, propositions per
 * position, '---' lines beyond the first), fill writes uint16[n][L] character matrices (zero beyond each length) and
 * the lengths.  Files not in canonical form (bytes other than 0 1 , ; - CR LF, ragged vectors, stray separators) are
 * refused with LTL_ERR_ARG and *bad_line = the 1-based line: the caller's line-by-line reader owns the messages. */
LTL_API int ltl_trace_file_scan(const char* data, uint64_t n, int64_t counts_out[2], int* max_len, int* width,
                                int* extra_sections, int64_t* bad_line);
LTL_API int ltl_trace_file_fill(const char* data, uint64_t n, int width, int L, uint16_t* pos_chars, int64_t* pos_lengths,
                                uint16_t* neg_chars, int64_t* neg_lengths);

/* Constructor: reference _speedups.pyx:79-111 (Core.__cinit__) / kernels.py:140-172 (make_core).
 * masks: uint64[R*W] length masks.  proj_rows/proj_offs (n_proj <= 126 pairs): gather projection
 * (row, position).  fkp_bits: per-row prefix width of the fkp variant.  mask_k: low fingerprint bits
 * cleared.  budget_bytes: logical budget, entry_bytes = 8*R*W + 16 (reference _speedups.pyx:100).
 * Differences by design: no R <= 64 limit, W up to 16 words per row. */
LTL_API int ltl_core_create(const uint64_t* masks, int R, int W, int n_pos, int err_max, int variant,
                    const int32_t* proj_rows, const int32_t* proj_offs, int n_proj, int fkp_bits, int mask_k,
                    uint64_t budget_bytes, int device, ltl_core** out);
LTL_API void ltl_core_destroy(ltl_core* h);
LTL_API const char* ltl_core_last_error(const ltl_core* h); /* h may be NULL: last create() failure */

/* add_entry: reference _speedups.pyx:264-277.  *index_out = new entry index, or -1 if the fingerprint is
 * already present.  Returns LTL_ERR_BUDGET where the reference raises CoreOOM.  No solve check. */
LTL_API int ltl_core_add_entry(ltl_core* h, const uint64_t* cm, int op, int lhs, int rhs, int64_t* index_out);

/* screen_unary / screen_binary: reference _speedups.pyx:337-355 / 357-380.  Candidates are treated
 * strictly in enumeration order; *status is LTL_S_*; (*li, *ri) are the solving operands or -1. */
LTL_API int ltl_core_screen_unary(ltl_core* h, int op, int64_t c0, int64_t c1, int* status, int64_t* li, int64_t* ri);
LTL_API int ltl_core_screen_binary(ltl_core* h, int op, int64_t a0, int64_t a1, int64_t b0, int64_t b1, int tri, int* status,
                           int64_t* li, int64_t* ri);

/* One whole cost level: the segment list of reference enumerator.py:271-296 (_run_level_core) in one call.
 * Equivalent to calling screen_* on every segment in order and stopping at the first status != DONE;
 * *seg_index is the segment of the solving candidate (or -1). */
LTL_API int ltl_core_run_level(ltl_core* h, const ltl_segment* segs, int n_segs, int* status, int* seg_index, int64_t* li,
                       int64_t* ri);

/* One whole search: the cost-level loop of reference enumerator.py:234-251 over a core whose atoms (and, for the NNF
 * fragment, negated atoms) are admitted -- per level the child-cost pairing of enumerator.py:254-268 (_bucket_pairs), the
 * dispatch order of enumerator.py:271-296 (connective order formula.py:24) and the bookkeeping of cache.py:144-166
 * (begin_level / end_level), i.e. exactly ltl_core_run_level on the segment list the reference would build, for
 * cost = first_cost .. ceiling - 1 until a level solves or runs out of memory.  Same results as the per-level calls;
 * what it removes is the caller's interpreter from between the levels (config 1: nine levels of a few hundred candidates).
 *   op_cost[8]     cost of each connective, indexed by opcode (reference formula.py:13-20; [0], the atom cost, is unused)
 *   op_mask        bit k set: connective k is enabled (NOT off for the NNF fragment, UNTIL off for forbid_until)
 *   bucket_*       the entry ranges admitted so far, by formula cost (atoms, negated atoms)
 *   store_last_level  0: entries of level ceiling - 1 keep records and fingerprints only (they are never operands)
 *   rows / n_rows  one row per level that ended (DONE or SOLVED), in order
 *   status, op, li, ri  outcome: LTL_S_DONE (ceiling reached), LTL_S_SOLVED with the solving connective and operands,
 *                  LTL_S_OOM, LTL_S_TIMEOUT; *end_cost = the level the search ended in (ceiling if none solved) */
typedef struct ltl_level_stats {
    int32_t cost, status;
    uint64_t offered, admitted, duplicates; /* of this level (reference cache.py:160-165) */
    uint64_t bytes;                         /* bytes_used after the level */
    int64_t first_entry, end_entry;         /* the level's bucket */
    double ms;                              /* host wall time of the level */
} ltl_level_stats;
LTL_API int ltl_core_run_search(ltl_core* h, const int32_t op_cost[8], uint32_t op_mask, const int64_t* bucket_cost,
                                const int64_t* bucket_first, const int64_t* bucket_end, int n_buckets, int first_cost,
                                int ceiling, int store_last_level, ltl_level_stats* rows, int max_rows, int* n_rows,
                                int* status, int* op, int64_t* li, int64_t* ri, int* end_cost);

/* contains / fingerprint_of: reference _speedups.pyx:279-287 / 233-241 (hi has its top 2 bits clear). */
LTL_API int ltl_core_contains(ltl_core* h, const uint64_t* cm, int* found);
LTL_API int ltl_core_fingerprint_of(ltl_core* h, const uint64_t* cm, uint64_t* hi, uint64_t* lo);

/* get_cm / get_record / export_cms: reference _speedups.pyx:117-137.  export_* copy entries
 * [first, first + count); cms_out is uint64[count][R*W] row-major. */
LTL_API int ltl_core_get_cm(ltl_core* h, int64_t idx, uint64_t* out);
LTL_API int ltl_core_get_record(ltl_core* h, int64_t idx, int* op, int* lhs, int* rhs);
/* The records of a whole formula in one call: every entry reachable from idx through (lhs, rhs), each once, idx first;
 * nodes = int32[cap][4] rows (entry, op, lhs, rhs).  What reference cache.py:197-213 (reconstruct) collects with one
 * get_record per node -- here one kernel and one copy instead of one device round trip per node. */
LTL_API int ltl_core_get_subtree(ltl_core* h, int64_t idx, int cap, int32_t* nodes, int* n_nodes);
LTL_API int ltl_core_export_cms(ltl_core* h, int64_t first, int64_t count, uint64_t* cms_out);
LTL_API int ltl_core_export_records(ltl_core* h, int64_t first, int64_t count, int8_t* op, int32_t* lhs, int32_t* rhs);

/* Fingerprints of stored entries [first, first + count) (set-parity checks; reference fingerprint_of over
 * export_cms). */
LTL_API int ltl_core_entry_fingerprints(ltl_core* h, int64_t first, int64_t count, uint64_t* hi, uint64_t* lo);

/* out[0..4] = n_entries, bytes_used, offered, admitted, duplicates: reference _speedups.pyx:68, 113-115. */
LTL_API int ltl_core_counters(ltl_core* h, uint64_t out[5]);

/* Row-sharded cores (the alternative for specifications with many rows): G cores, one per GPU, each
 * created over a contiguous slice of the ROWS of the specification (masks of its rows, n_pos = its number of
 * positive rows).  Every core enumerates every candidate on its rows; the per-candidate partial fingerprint sums and
 * error counts -- a device array of 3 uint64 per candidate, (s0, s1, errors) -- are handed to `fn`, which must
 * replace them by their element-wise sums over all shards (wrapping 64-bit adds; ONE NCCL all-reduce of 3 * count
 * int64) and return 0 once the result is visible to the device; every core then completes identical candidates, admits
 * the same entries in the same order and writes its rows of the new matrices.  A pass is handed over in up to
 * "exchange_parts" (option, default 4) consecutive candidate ranges: `fn` is called for a range as soon as its
 * evaluation has ended on the device while the next range is still being evaluated on the core's stream, so the
 * all-reduce (on the caller's stream) overlaps phase A.  No reference counterpart (the reference is one process); the
 * results are those of one core over all rows.
 * word_base: index of this shard's first word in the whole matrix (rows before it x W), a multiple of 64;
 * total_words: words of the whole matrix (the budget counts whole matrices: reference _speedups.pyx:100, 252-253).
 * Call once, right after ltl_core_create.  Needs a block-combinable fingerprint (LTL_V_MUELLER / LTL_V_NH / LTL_V_NH32). */
typedef int (*ltl_exchange_fn)(void* ctx, void* d_sums, int64_t count);
LTL_API int ltl_core_set_row_shard(ltl_core* h, int64_t word_base, int64_t total_words, ltl_exchange_fn fn, void* ctx);
/* Optional, right after ltl_core_set_row_shard: shard the uniqueness table as well.  Core `shard` of `n_shards` then
 * files only the candidates whose fingerprint it owns (owner = mix(hi ^ lo) mod n_shards, the rule of the
 * candidate-range shards), the winner flags -- one bit per candidate, set by one shard at most -- are OR-ed over the
 * shards through `fn` (a wrapping sum of disjoint bits), and every core compacts the same winners.  The table's memory
 * and the work of filing keys then scale with the number of GPUs like everything else; results are unchanged. */
LTL_API int ltl_core_set_table_shard(ltl_core* h, int shard, int n_shards);

/* Tuning / measurement (no reference counterpart).
 * options: "deadline_ms" (run_level / screen_* return LTL_S_TIMEOUT at the first pass boundary more than this many
 * milliseconds from now; 0 disarms), "chunk_candidates" (candidates per device pass), "profile" (1: time every kernel with CUDA
 * events on the launching stream), "max_split" (cap on row splits), "force_split" (tests),
 * "store_results" (0: from now on admitted entries keep fingerprint + record but their matrices are not
 * written -- for the last cost level of a search, whose entries are never operands; counters, records and
 * statuses are unaffected, get_cm / export_cms of such entries fail with LTL_ERR_ARG),
 * "gate_store" (default 1: the phase B that also screens NOT(new entry) is issued behind the level's phase A and writes
 * the matrices only if that found no solver; 0: always write first, the order of round 1). */
LTL_API int ltl_core_set_option(ltl_core* h, const char* name, int64_t value);
/* Accumulated per kernel class since creation / the last reset: launches, device milliseconds (profile
 * mode only), algorithmic bytes and candidates / entries processed. */
LTL_API int ltl_core_kernel_stats(ltl_core* h, int kernel_class, uint64_t* launches, double* ms, double* alg_bytes,
                          uint64_t* units);
LTL_API int ltl_core_reset_kernel_stats(ltl_core* h);
/* The CUDA stream (cudaStream_t) every kernel and copy of this handle is issued on, for CUDA-event timing. */
LTL_API int ltl_core_stream(ltl_core* h, void** stream_out);
/* ---- Multi-GPU stages (one process per GPU; orchestration in paper_2402_12373_b200/sharded.py). ----------
 * A cost level's candidates have level ranks 0 .. level_size-1 in enumeration order; every rank of the job
 * holds the same replicated store and evaluates a contiguous slice.  d_* arguments are DEVICE pointers on the
 * handle's device (torch tensors); every stage returns after its work completed on the device.
 *   level_size   candidates in the level
 *   stage_eval   fingerprints (hi, lo per candidate, 2 x uint64) of level ranks [lo, hi) and the lowest
 *                solving level rank in the slice (-1: none); stops after the chunk that holds a solver
 *   stage_file   owner side: file (hi, lo, global rank) tuples in this handle's table shard with
 *                atomicMin(rank); d_win[t] = 1 iff tuple t owns its key and the key was not a member before
 *   stage_route  (hi, lo) fingerprints of level ranks rank_base .. -> (hi, lo, global rank) tuples grouped by owner
 *                rank = mix(hi ^ lo) mod world (in rank order inside a group: a stable counting sort on the device),
 *                and the number of tuples per owner -- the send buffer and split sizes of the all-to-all
 *   stage_winners  the owners' verdict bytes, in the order the tuples were sent -> the level ranks of this slice's
 *                winners, ascending (device array d_out of at least `count` int64), and how many there are
 *   stage_decode level ranks -> (op, lhs, rhs) records
 *   stage_append append `count` admitted entries (records, in rank order) and advance the counters;
 *                matrices are materialised locally from the records when first needed
 *   stage_purge  forget keys filed at or above a global rank (solver / budget cut) */
LTL_API int ltl_core_level_size(ltl_core* h, const ltl_segment* segs, int n_segs, int64_t* total);

/* The planner of the device-resident cost levels, callable on the host (no GPU, no handle): the pieces of cost level
 * `cost` in enumeration order -- what ltl_core_run_search's first launch (csrc/levels.cuh) builds for itself on the device
 * from its bucket table, i.e. the child-cost pairing of reference enumerator.py:254-268 in the dispatch order of 271-296
 * with triangular segments expanded as _speedups.pyx:364-368 does.  Buckets as for ltl_core_run_search.  Per piece:
 * op_out, kind_out (0 unary [i0, i1); 1 rectangle [i0, i1) x [j0, j1); 2 triangle i in [i0, i1), j in (i, j1)),
 * range_out[4] = i0, i1, j0, j1 and count_out.  Returns LTL_ERR_ARG when the level needs more than `cap` pieces. */
LTL_API int ltl_plan_level(const int32_t op_cost[8], uint32_t op_mask, const int64_t* bucket_cost, const int64_t* bucket_first,
                           const int64_t* bucket_end, int n_buckets, int cost, int cap, int32_t* op_out, int32_t* kind_out,
                           int64_t* range_out, int64_t* count_out, int* n_pieces, int64_t* total);
LTL_API int ltl_core_stage_eval(ltl_core* h, const ltl_segment* segs, int n_segs, int64_t lo, int64_t hi, uint64_t* d_fp,
                        int64_t* solver_rank);
LTL_API int ltl_core_stage_file(ltl_core* h, const uint64_t* d_tuples, int64_t count, unsigned char* d_win, int64_t* n_win);
LTL_API int ltl_core_stage_route(ltl_core* h, const uint64_t* d_fp, int64_t count, uint64_t rank_base, int world,
                                 uint64_t* d_send, int64_t* counts_out);
LTL_API int ltl_core_stage_winners(ltl_core* h, const uint64_t* d_tuples, const unsigned char* d_win, int64_t count,
                                   uint64_t rank_base, int64_t level_lo, int64_t* d_out, int64_t* n_out);
LTL_API int ltl_core_stage_decode(ltl_core* h, const ltl_segment* segs, int n_segs, const int64_t* d_ranks, int64_t count,
                          unsigned char* d_op, int32_t* d_lhs, int32_t* d_rhs);
LTL_API int ltl_core_stage_append(ltl_core* h, const unsigned char* d_op, const int32_t* d_lhs, const int32_t* d_rhs,
                          int64_t count, uint64_t offered_delta, uint64_t duplicates_delta);
LTL_API int ltl_core_stage_purge(ltl_core* h, uint64_t global_rank_cut);

/* Released stores are pooled per process (virtual range + physical pages) for the next core; this returns
 * every pooled page to the driver and reports the bytes freed.  LTL_NO_POOL=1 disables pooling. */
LTL_API uint64_t ltl_pool_trim(void);
/* out[0..2] = host wall milliseconds spent growing the store, waiting for the device, planning chunks. */
LTL_API int ltl_core_host_times(ltl_core* h, double out[3]);
/* out[0..1] = bytes copied host->device / device->host by this handle so far. */
LTL_API int ltl_core_transfer_stats(ltl_core* h, uint64_t out[2]);
/* out[0..5] = effective entry capacity, device bytes mapped for matrices, table slots, chunk candidates,
 * bit 0: the store uses virtual-memory growth, bit 1: an S_OOM status came from exhausted DEVICE memory rather
 * than from the logical budget, bits 8..: conditional phase-B launches that skipped their store because the pass they
 * were issued behind had found a solver (option "gate_store"); words per matrix */
LTL_API int ltl_core_info(ltl_core* h, uint64_t out[6]);

#ifdef __cplusplus
}
#endif
#endif /* LTL_CORE_H */
