// levels.cuh -- device-resident cost levels: the level loop of a search, for as long as the levels are small, in ONE
// kernel launch (a thread-block cluster of 1024-thread CTAs; hardware cluster barriers between the phases of a level).
//
// A cost level of a few hundred candidates costs the host-driven path three launches and one host round trip, ~55 us
// whatever the work: BASELINE config 1 (16 traces, 5,762 candidates over six levels) spent 0.74 ms per search of which
// 0.32 ms were kernels.  Here the device plans a level's pieces itself (the child-cost pairing of reference
// enumerator.py:254-268 in the dispatch order of 271-296, from the bucket table it keeps), screens the candidates
// (small_rows: same connectives, same fingerprints, same table filing as every other phase-A kernel), admits the winners
// in rank order (the k_admit_small scheme), writes their records and matrices, closes the level (cache.py:154-166) and
// goes on, until a level solves, is too large for one cluster, or could run out of budget / table / store -- that level
// and everything after it is run by the host-driven path (ltl_core_run_search), which continues from the state left
// here.  Results are bit-identical to the host-driven path: same ranks, same winners, same entry order and records.
#pragma once
#include "screen.cuh"

#define LTL_LV_MAX_COST 64    // cost levels (and bucket table entries) a launch can see
#define LTL_LV_MAX_PIECES 96
#define LTL_LV_CTA 1024
#define LTL_LV_MAX_CLUSTER 8  // portable cluster size
#define LTL_LV_MAX_TOTAL 32768  // candidates per level (scratch arrays; one CTA admits 1024 per ~1.5 us round)

struct LevelRow {
    int cost, status;
    u64 offered, admitted, duplicates;
    i64 first_entry, end_entry;
};

// Device-resident search state; the host fills it before the launch and reads it back once afterwards.
struct LevelsState {
    u64 n_entries, offered, admitted, duplicates, keys_upper;
    int next_cost;  // the first cost level this launch did NOT complete (== the solved level when status is SOLVED)
    int status;     // LTL_S_DONE / LTL_S_SOLVED
    int sol_op, n_rows;
    i64 sol_li, sol_ri;
    u64 sol_cut, sol_gbase;        // solved level: chunk-local rank of the solver, global rank of the level's first candidate
    u64 pend_base, pend_count;     // solved level: admitted entries whose records exist and whose matrices do not
    u64 lv_count, lv_solver;       // the level in flight: winners below the cut, rank of the first solver (~0: none)
    u64 unstored_from;             // first entry without a matrix (the unstored last level admitted something), else ~0
    double alg_bytes;              // algorithmic bytes of the candidates screened
    i64 bucket_first[LTL_LV_MAX_COST], bucket_end[LTL_LV_MAX_COST];
    int known[LTL_LV_MAX_COST];
    LevelRow rows[LTL_LV_MAX_COST];
    u64 t_ns[LTL_LV_MAX_COST][6];  // %globaltimer of CTA 0 per completed level: start, planned, screened, admitted, booked, stored
};

struct LevelsParams {
    ScreenParams sp;  // store, masks, shape, fingerprint variant, table, slot / acc scratch, ctl; mode INSERT, check_solve
    u64* cms_w;       // the store, writable
    unsigned char* rec_op;
    int* rec_lhs;
    int* rec_rhs;
    LevelsState* st;
    int first_cost, stop_cost;  // levels [first_cost, stop_cost)
    int nostore_cost;           // the level whose winners get no matrices (the last level of a search), or -1
    int op_cost[8];
    u32 op_mask;
    i64 max_total;   // candidates per level the scratch arrays hold
    i64 max_work;    // candidate-words per level worth running on one cluster
    u64 entry_cap;   // entries the store and the budget have room for (absolute)
    u64 table_cap;   // slots of the uniqueness table
};

// The pieces of cost level c in enumeration order (segments of ltl_core_run_search expanded as expand_segments does).
// Returns false when the level has more pieces than `cap`.
template <bool FULL = true>  // false: only the fields the small-pass kernels read (op, kind, ranges, cbase, count)
__host__ __device__ inline bool lv_plan(const int c, const int* op_cost, const u32 op_mask, const i64* bfirst, const i64* bend,
                                        Piece* pieces, const int cap, int* np_out, i64* total_out, double* bytes_out,
                                        const double B) {
    const int ORDER[7] = {OP_NOT, OP_AND, OP_OR, OP_NEXT, OP_FINALLY, OP_GLOBALLY, OP_UNTIL};  // reference formula.py:24
    int np = 0, seg = 0;
    i64 total = 0;
    double bytes = 0;
    auto push = [&](int op, int kind, i64 i0, i64 i1, i64 j0, i64 j1) -> bool {
        if (np >= cap) return false;
        Piece& p = pieces[np];
        p.op = op;
        p.kind = kind;
        if (FULL) {
            p.swap = 0;
            p.ti = 1;
            p.seg = seg;
            p.owns_tiles = 1;
            p.ext = 0;
            p.pad_ = 0;
            p.tile_base = p.tiles_lane = p.tiles_row = p.lane_g0 = 0;
            p.nfuse = 0;
            p.fops = 0;
            p.fcbase[0] = p.fcbase[1] = p.fcbase[2] = p.fcbase[3] = 0;
        }
        p.i0 = i0;
        p.i1 = i1;
        p.j0 = j0;
        p.j1 = j1;
        p.cbase = total;
        p.count = kind == PIECE_UNARY ? i1 - i0 : kind == PIECE_RECT ? (i1 - i0) * (j1 - j0) : (i64)tri_before((u64)(i1 - i0), (u64)(j1 - 1 - i0));
        total += p.count;
        bytes += (double)p.count * ((kind == PIECE_UNARY ? 1.0 : 2.0) * B + 16.0);
        np++;
        return true;
    };
    for (int oi = 0; oi < 7; oi++) {
        const int o = ORDER[oi];
        if (!((op_mask >> o) & 1u)) continue;
        const int w = op_cost[o];
        if (o == OP_NOT || o == OP_NEXT || o == OP_FINALLY || o == OP_GLOBALLY) {
            const int a = c - w;
            if (a >= 1 && a < LTL_LV_MAX_COST && bend[a] > bfirst[a]) {
                if (!push(o, PIECE_UNARY, bfirst[a], bend[a], -1, -1)) return false;
                seg++;
            }
            continue;
        }
        const bool commutative = o == OP_AND || o == OP_OR;
        for (int a = 1; a < c - w; a++) {
            const int b = c - w - a;
            if (b < 1) continue;
            if (commutative && a > b) break;
            if (a >= LTL_LV_MAX_COST || b >= LTL_LV_MAX_COST) continue;
            const i64 a0 = bfirst[a], a1 = bend[a], b0 = bfirst[b], b1 = bend[b];
            if (a1 == a0 || b1 == b0) continue;
            if (!(commutative && a == b)) {
                if (!push(o, PIECE_RECT, a0, a1, b0, b1)) return false;
            } else {  // unordered pairs i < j of one bucket
                const i64 rect_end = a1 < b0 ? a1 : b0;
                if (a0 < rect_end && !push(o, PIECE_RECT, a0, rect_end, b0, b1)) return false;
                const i64 t0 = a0 > b0 ? a0 : b0, t1 = a1 < b1 - 1 ? a1 : b1 - 1;
                if (t0 < t1 && !push(o, PIECE_TRI, t0, t1, -1, b1)) return false;
            }
            seg++;
        }
    }
    *np_out = np;
    *total_out = total;
    *bytes_out = bytes;
    return true;
}

// May cost level c, of `total` candidates in `np` pieces, run inside the launch?  (No: the host-driven path takes over.)
__host__ __device__ inline bool lv_fits(const LevelsParams& P, const i64 total, const u64 n_entries, const u64 keys_upper) {
    if (total > P.max_total || total * (i64)P.sp.R > P.max_work) return false;
    if (n_entries + (u64)total > P.entry_cap) return false;                   // could run out of budget or store
    if ((keys_upper + (u64)total) * 2 > P.table_cap) return false;            // the table would have to grow first
    return true;
}

#ifdef __CUDACC__

__device__ __forceinline__ u64 lv_now() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ u32 lv_cluster_rank() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ u32 lv_cluster_size() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// all threads of all CTAs of the cluster; writes before it (global memory included) are visible after it
__device__ __forceinline__ void lv_sync() {
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int KIND>
__global__ void __launch_bounds__(LTL_LV_CTA, 1) k_levels(const __grid_constant__ LevelsParams P) {
    constexpr bool HASHED = KIND == KIND_NH || KIND == KIND_MUELLER;
    __shared__ Piece pieces[LTL_LV_MAX_PIECES];
    __shared__ ScreenParams s_p;  // the level's screening parameters (what a host-driven pass gets as its kernel argument)
    // every CTA keeps its own copy of the search state and moves it on from the two words CTA 0 publishes per level
    // (winners, solver rank): planning a level needs no global load
    __shared__ i64 s_bf[LTL_LV_MAX_COST], s_be[LTL_LV_MAX_COST];
    __shared__ int s_known[LTL_LV_MAX_COST];
    __shared__ u64 s_entries, s_offered, s_keys, s_admitted, s_dups;
    __shared__ int s_np, s_go, s_rows;
    __shared__ i64 s_total;
    __shared__ double s_bytes;
    __shared__ u32 wcnt[32];
    __shared__ u64 carry_s;
    const u32 rank = lv_cluster_rank();
    const i64 gt = (i64)rank * LTL_LV_CTA + threadIdx.x, gstride = (i64)lv_cluster_size() * LTL_LV_CTA;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    LevelsState* const st = P.st;
    const i64 n = P.sp.n;
    const int R = P.sp.R;
    const int nblk = (R + LTL_SPLIT_ROWS - 1) / LTL_SPLIT_ROWS;
    const ScreenParams& p = s_p;

    if (threadIdx.x < LTL_LV_MAX_COST) {
        s_bf[threadIdx.x] = st->bucket_first[threadIdx.x];
        s_be[threadIdx.x] = st->bucket_end[threadIdx.x];
        s_known[threadIdx.x] = st->known[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        s_entries = st->n_entries;
        s_offered = st->offered;
        s_keys = st->keys_upper;
        s_admitted = st->admitted;
        s_dups = st->duplicates;
        s_rows = 0;
        s_p = P.sp;
        s_p.pieces = pieces;
        s_p.nsplit = nblk;
        s_p.rows_per_split = LTL_SPLIT_ROWS;
    }
    __syncthreads();

    int c = P.first_cost;
    for (;; c++) {
        // ---- phase 0: every CTA plans the level (identical results everywhere)
        const bool clk = rank == 0 && threadIdx.x == 0;
        u64 t0 = 0, t1 = 0, t2 = 0, t3 = 0;
        if (clk) t0 = lv_now();
        if (threadIdx.x == 0) {
            int go = c < P.stop_cost;
            int np = 0;
            i64 total = 0;
            double bytes = 0;
            if (go)
                go = lv_plan<false>(c, P.op_cost, P.op_mask, s_bf, s_be, pieces, LTL_LV_MAX_PIECES, &np, &total, &bytes, 8.0 * (double)n) &&
                     lv_fits(P, total, s_entries, s_keys);
            s_go = go;
            s_np = np;
            s_total = total;
            s_bytes = bytes;
            s_p.n_pieces = np;
            s_p.gbase = s_offered;
        }
        __syncthreads();
        if (!s_go) break;
        const i64 total = s_total;
        const int np = s_np;
        const u64 n0 = s_entries;
        if (clk) t1 = lv_now();

        // ---- phase 1: screen.  One work item = (candidate, block of 64 rows), candidates fastest: neighbouring threads
        // share the left operand and read neighbouring right operands.  NH: 8 lanes per item (small_block_nh8); the
        // sequential fingerprints (Mueller, deposits): one thread per item
        if (KIND == KIND_NH) {
            const i64 items = total * nblk, nw = gstride >> 5;
            for (i64 base = (gt >> 5) * 4; base < items; base += nw * 4) {  // (warp-uniform trip count: the lanes shuffle)
                const i64 it = base + (lane >> 3);
                const bool valid = it < items;
                u64 cnd = 0;
                int op = 0, r0 = 0;
                const u64 *px = p.cms, *py = p.cms;
                if (valid) {
                    const i64 b = it / total;
                    cnd = (u64)(it - b * total);
                    int lo = 0, hi = np - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if ((u64)pieces[mid].cbase <= cnd) lo = mid;
                        else hi = mid - 1;
                    }
                    i64 i, j;
                    piece_unrank(pieces[lo], cnd, &i, &j);
                    op = pieces[lo].op;
                    px = p.cms + cm_index(i, n, 0);
                    py = j >= 0 ? p.cms + cm_index(j, n, 0) : px;
                    r0 = (int)b * LTL_SPLIT_ROWS;
                }
                u64 s0, s1;
                u32 err;
                small_block_nh8<false>(p, op, px, py, r0, min(R, r0 + LTL_SPLIT_ROWS), lane & 7, valid, s0, s1, err);
                if (!valid || (lane & 7)) continue;
                if (nblk == 1) {
                    finish_candidate<HASHED>(p, cnd, s0, s1, err);
                } else {
                    atomicAdd(p.acc + 3 * cnd, s0);
                    atomicAdd(p.acc + 3 * cnd + 1, s1);
                    if (err) atomicAdd(p.acc + 3 * cnd + 2, (u64)err);
                }
            }
        } else {
            for (i64 it = gt; it < total * nblk; it += gstride) {
                const i64 b = it / total;
                const u64 cnd = (u64)(it - b * total);
                int lo = 0, hi = np - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if ((u64)pieces[mid].cbase <= cnd) lo = mid;
                    else hi = mid - 1;
                }
                i64 i, j;
                piece_unrank(pieces[lo], cnd, &i, &j);
                const u64* px = p.cms + cm_index(i, n, 0);
                const u64* py = j >= 0 ? p.cms + cm_index(j, n, 0) : px;
                const int r0 = (int)b * LTL_SPLIT_ROWS, r1 = min(R, r0 + LTL_SPLIT_ROWS);
                u64 s0 = 0, s1 = 0;
                u32 err = 0;
                small_rows<KIND, false, 4>(p, pieces[lo].op, px, py, r0, r1, s0, s1, err);
                if (nblk == 1) {
                    finish_candidate<HASHED>(p, cnd, s0, s1, err);
                } else {
                    atomicAdd(p.acc + 3 * cnd, s0);
                    atomicAdd(p.acc + 3 * cnd + 1, s1);
                    if (err) atomicAdd(p.acc + 3 * cnd + 2, (u64)err);
                }
            }
        }
        lv_sync();
        if (nblk > 1) {  // complete the candidates from their blocks' sums; the sums go back to zero
            for (i64 cnd = gt; cnd < total; cnd += gstride) {
                const u64 s0 = __ldcg(p.acc + 3 * cnd), s1 = __ldcg(p.acc + 3 * cnd + 1), er = __ldcg(p.acc + 3 * cnd + 2);
                finish_candidate<HASHED>(p, (u64)cnd, s0, s1, (u32)er);
                p.acc[3 * cnd] = 0;
                p.acc[3 * cnd + 1] = 0;
                p.acc[3 * cnd + 2] = 0;
            }
            lv_sync();
        }

        // ---- phase 2 (CTA 0): ordered admission (the k_admit_small scheme) and the winners' records
        if (clk) t2 = lv_now();
        if (rank == 0) {
            if (threadIdx.x == 0) carry_s = 0;
            __syncthreads();
            const u64 solver = __ldcg(&p.ctl->solver_c);
            const u64 limit = min((u64)total, solver);  // nothing at or above the first solver is admitted
            for (u64 base = 0; base < limit; base += LTL_LV_CTA) {
                const u64 cnd = base + threadIdx.x;
                bool win = false;
                if (cnd < limit) {
                    const u32 s = __ldcg(p.slot + cnd);
                    if (s != LTL_NONE) win = ld_rank(p.table + s) == p.gbase + cnd;
                }
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, win);
                if (lane == 0) wcnt[warp] = __popc(bal);
                __syncthreads();
                u64 dest = carry_s + __popc(bal & ((1u << lane) - 1u));
                u32 block_total = 0;
                for (int w = 0; w < 32; w++) {
                    const u32 v = wcnt[w];
                    if (w < warp) dest += v;
                    block_total += v;
                }
                if (win) {
                    int lo = 0, hi = np - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if ((u64)pieces[mid].cbase <= cnd) lo = mid;
                        else hi = mid - 1;
                    }
                    i64 i, j;
                    piece_unrank(pieces[lo], cnd, &i, &j);
                    const i64 e = (i64)n0 + (i64)dest;
                    P.rec_op[e] = (unsigned char)pieces[lo].op;
                    P.rec_lhs[e] = (int)i;
                    P.rec_rhs[e] = (int)j;
                }
                __syncthreads();
                if (threadIdx.x == 0) carry_s += block_total;
                __syncthreads();
            }
            if (threadIdx.x == 0) {  // publish the outcome; re-arm the solver word for the next level
                st->lv_count = carry_s;
                st->lv_solver = solver;
                p.ctl->solver_c = ~0ull;
            }
        }
        lv_sync();

        // ---- the level's bookkeeping, in every CTA's copy of the state (reference cache.py:154-166; counters:
        // _speedups.pyx:347-354, 372-379); CTA 0 also writes the stats row
        const u64 count = __ldcg(&st->lv_count), solver = __ldcg(&st->lv_solver);
        const bool solved = solver != ~0ull;
        if (clk) t3 = lv_now();
        __syncthreads();  // (every thread has read the shared state of phase 0)
        if (threadIdx.x == 0) {
            const u64 offered_c = solved ? solver + 1 : (u64)total;
            const u64 dups = (solved ? solver : (u64)total) - count;
            const i64 first = s_known[c] ? s_bf[c] : (i64)n0;  // a bucket that exists already (negated atoms, NNF) grows
            s_bf[c] = first;
            s_be[c] = (i64)(n0 + count);
            s_known[c] = 1;
            const u64 gbase = s_offered;
            s_offered = gbase + offered_c;
            s_admitted += count;
            s_dups += dups;
            s_entries = n0 + count;
            s_keys += solved ? (u64)total : count;  // keys filed above the cut stay until the purge
            if (rank == 0) {
                LevelRow& row = st->rows[s_rows];
                row.cost = c;
                row.status = solved ? LTL_S_SOLVED : LTL_S_DONE;
                row.offered = offered_c;
                row.admitted = count;
                row.duplicates = dups;
                row.first_entry = first;
                row.end_entry = (i64)(n0 + count);
                s_rows++;
                double done = s_bytes;
                if (solved) {  // algorithmic bytes of the candidates that were screened: up to the cut, like the host-driven path
                    done = 0;
                    const double B = 8.0 * (double)n;
                    for (int k = 0; k < np; k++) {
                        const i64 upto = min(pieces[k].count, max((i64)0, (i64)offered_c - pieces[k].cbase));
                        done += (double)upto * ((pieces[k].kind == PIECE_UNARY ? 1.0 : 2.0) * B + 16.0);
                    }
                    int lo = 0, hi = np - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if ((u64)pieces[mid].cbase <= solver) lo = mid;
                        else hi = mid - 1;
                    }
                    i64 i, j;
                    piece_unrank(pieces[lo], solver, &i, &j);
                    st->sol_op = pieces[lo].op;
                    st->sol_li = i;
                    st->sol_ri = j;
                    st->sol_cut = solver;
                    st->sol_gbase = gbase;
                    st->pend_base = n0;
                    st->pend_count = count;
                    st->status = LTL_S_SOLVED;
                }
                st->alg_bytes += done;
                if (c == P.nostore_cost && count > 0) st->unstored_from = n0;
                u64* tn = st->t_ns[s_rows - 1];
                tn[0] = t0;
                tn[1] = t1;
                tn[2] = t2;
                tn[3] = t3;
                tn[4] = lv_now();
                tn[5] = 0;
            }
        }
        if (solved) break;  // a search that ends here never pays for the matrices
        if (c == P.nostore_cost) {  // the last level of a search: records and fingerprints, no matrices
            __syncthreads();
            continue;
        }

        // ---- phase 3: the winners' matrices, from their records.  One work item = (entry, block of 64 rows) for 8 lanes
        // (lane `sub`: rows sub, sub + 8, ...; four loads in flight each), entries fastest
        for (i64 it = gt >> 3; it < (i64)count * nblk; it += gstride >> 3) {
            const int sub = lane & 7;
            const i64 b = it / (i64)count;
            const i64 e = (i64)n0 + (it - b * (i64)count);
            const int op = (int)__ldcg(P.rec_op + e);
            const i64 lhs = __ldcg(P.rec_lhs + e), rhs = __ldcg(P.rec_rhs + e);
            const u64* px = p.cms + cm_index(lhs, n, 0);
            const u64* py = rhs >= 0 ? p.cms + cm_index(rhs, n, 0) : px;
            u64* po = P.cms_w + cm_index(e, n, 0);
            const int r0 = (int)b * LTL_SPLIT_ROWS, r1 = min(R, r0 + LTL_SPLIT_ROWS);
#pragma unroll
            for (int half = 0; half < 2; half++) {
                u64 xv[4], yv[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int r = r0 + sub + 8 * (4 * half + k);
                    xv[k] = r < r1 ? __ldcg(px + (size_t)r * 32) : 0ull;
                    yv[k] = r < r1 && rhs >= 0 ? __ldcg(py + (size_t)r * 32) : 0ull;
                }
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int r = r0 + sub + 8 * (4 * half + k);
                    if (r < r1) po[(size_t)r * 32] = small_apply(op, xv[k], yv[k], ld_nc(p.masks + r));
                }
            }
        }
        lv_sync();
        if (clk) st->t_ns[s_rows - 1][5] = lv_now();
    }
    // ---- the state the host-driven path continues from
    __syncthreads();
    if (rank == 0) {
        if (threadIdx.x < LTL_LV_MAX_COST) {
            st->bucket_first[threadIdx.x] = s_bf[threadIdx.x];
            st->bucket_end[threadIdx.x] = s_be[threadIdx.x];
            st->known[threadIdx.x] = s_known[threadIdx.x];
        }
        if (threadIdx.x == 0) {
            st->n_entries = s_entries;
            st->offered = s_offered;
            st->admitted = s_admitted;
            st->duplicates = s_dups;
            st->keys_upper = s_keys;
            st->n_rows = s_rows;
            st->next_cost = c;
        }
    }
}

#endif  // __CUDACC__
