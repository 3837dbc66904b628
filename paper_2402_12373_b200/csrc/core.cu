// core.cu -- host side of the B200 screening core + the small bookkeeping kernels + the C ABI
// (include/ltl_core.h).  The two hot kernels live in screen.cuh.
//
// One "chunk" (<= chunk_candidates candidates, consecutive in enumeration order) runs as
//   k_screen      every candidate: evaluate, count errors, fingerprint, claim its table slot with
//                 atomicMin(rank)                                   (reference _speedups.pyx:364-379)
//   k_resolve     a candidate is admitted iff its rank is the one left in the slot  (first-wins)
//   k_scan/k_emit ordered compaction: winners get consecutive entry indices in rank order and their
//                 (op, lhs, rhs) records                            (reference _speedups.pyx:255-262)
//   k_materialize winners' matrices are re-evaluated and appended to the store
// so that entry order, records and counters equal the sequential reference's.
#include <cuda.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ltl_core.h"
#include "screen.cuh"
#include "levels.cuh"
#include "traces.cuh"

// ------------------------------------------------------------------------------------------------
// per-W launchers (screen_inst.cu)

#define LTL_MAX_DEVICES 64

#define LTL_DECL_W(N)                                                                                  \
    extern "C" void ltl_launch_screen_w##N(const ScreenParams&, int, dim3, cudaStream_t);             \
    extern "C" void ltl_launch_materialize_w##N(const MaterializeParams&, const ScreenParams&, int, dim3, cudaStream_t);
LTL_DECL_W(1) LTL_DECL_W(2) LTL_DECL_W(3) LTL_DECL_W(4) LTL_DECL_W(5) LTL_DECL_W(6) LTL_DECL_W(7) LTL_DECL_W(8)
LTL_DECL_W(9) LTL_DECL_W(10) LTL_DECL_W(11) LTL_DECL_W(12) LTL_DECL_W(13) LTL_DECL_W(14) LTL_DECL_W(15) LTL_DECL_W(16)
#undef LTL_DECL_W
// half-width store (two 32-bit rows per word): screen_inst.cu compiled with -DLTL_W=1 -DLTL_PAIR
extern "C" void ltl_launch_screen_w1p(const ScreenParams&, int, dim3, cudaStream_t);
extern "C" void ltl_launch_screen_small(const ScreenParams&, int, unsigned long long, cudaStream_t);
extern "C" void ltl_launch_materialize_w1p(const MaterializeParams&, const ScreenParams&, int, dim3, cudaStream_t);
// small NH passes over rows of 2 / 4 / 8 / 16 words
extern "C" void ltl_launch_screen_small_w2(const ScreenParams&, unsigned long long, cudaStream_t);
extern "C" void ltl_launch_screen_small_w4(const ScreenParams&, unsigned long long, cudaStream_t);
extern "C" void ltl_launch_screen_small_w8(const ScreenParams&, unsigned long long, cudaStream_t);
extern "C" void ltl_launch_screen_small_w16(const ScreenParams&, unsigned long long, cudaStream_t);

static const screen_launch_fn SCREEN_FN[LTL_MAX_W + 1] = {
    nullptr, ltl_launch_screen_w1, ltl_launch_screen_w2, ltl_launch_screen_w3, ltl_launch_screen_w4,
    ltl_launch_screen_w5, ltl_launch_screen_w6, ltl_launch_screen_w7, ltl_launch_screen_w8, ltl_launch_screen_w9,
    ltl_launch_screen_w10, ltl_launch_screen_w11, ltl_launch_screen_w12, ltl_launch_screen_w13,
    ltl_launch_screen_w14, ltl_launch_screen_w15, ltl_launch_screen_w16};
static const materialize_launch_fn MATERIALIZE_FN[LTL_MAX_W + 1] = {
    nullptr, ltl_launch_materialize_w1, ltl_launch_materialize_w2, ltl_launch_materialize_w3,
    ltl_launch_materialize_w4, ltl_launch_materialize_w5, ltl_launch_materialize_w6, ltl_launch_materialize_w7,
    ltl_launch_materialize_w8, ltl_launch_materialize_w9, ltl_launch_materialize_w10, ltl_launch_materialize_w11,
    ltl_launch_materialize_w12, ltl_launch_materialize_w13, ltl_launch_materialize_w14, ltl_launch_materialize_w15,
    ltl_launch_materialize_w16};

// ------------------------------------------------------------------------------------------------
// bookkeeping kernels

#define RES_CTA 1024

template <bool MUELLER>
__global__ void k_finalize(const __grid_constant__ ScreenParams p, u64 total) {
    u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= total) return;
    finish_candidate<MUELLER>(p, c, p.acc[3 * c], p.acc[3 * c + 1], (u32)p.acc[3 * c + 2]);
}

// ------------------------------------------------------------------------------------------------
// trace packing (reference bitsem.py:73-88, TraceContext.from_traces; layout rule N2)
//
// One thread per (row, word): 64 consecutive characters of the row (128 contiguous bytes, read as eight 16-byte
// vectors) become one word of the length mask and one word of every proposition's characteristic sequence --
// position j at bit 63 - j%64, positions >= length zero.  Outputs are row-major [R, W] per proposition.
template <int NP>
__global__ void __launch_bounds__(256) k_pack(const uint16_t* __restrict__ chars, const i64* __restrict__ lengths, i64 R, int L,
                                             int Lpad, int W, int n_props, u64* __restrict__ masks, u64* __restrict__ atoms) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R * W) return;
    const i64 r = t / W;
    const int w = (int)(t - r * W);
    const i64 len64 = lengths[r];
    const int len = len64 < (i64)L ? (int)len64 : L;
    const int j0 = w * 64;
    const int live = max(0, min(64, len - j0));
    u64 acc[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) acc[p] = 0;
    const uint16_t* row = chars + (size_t)r * Lpad + j0;
    for (int v = 0; v < 8 && v * 8 < live; v++) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(row) + v);  // Lpad is a multiple of 64: always in bounds
        const u32 c[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int j = v * 8 + k;
            const u32 ch = (c[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
            if (j < live) {
#pragma unroll
                for (int p = 0; p < NP; p++)
                    if (p < n_props) acc[p] |= (u64)((ch >> p) & 1u) << (63 - j);
            }
        }
    }
    masks[t] = live == 0 ? 0ull : (~0ull << ((64 - live) & 63));  // live = 64: shift by 0
    for (int p = 0; p < NP; p++)
        if (p < n_props) atoms[(size_t)p * (size_t)(R * W) + (size_t)t] = acc[p];
}

// winner flags (one bit per candidate) + winners per 1024-candidate block
__global__ void __launch_bounds__(RES_CTA) k_resolve(const u32* __restrict__ slot, const Slot* __restrict__ table,
                                                     u64 gbase, u64 total, const Ctl* __restrict__ ctl,
                                                     u32* __restrict__ flagw, u32* __restrict__ blocksum) {
    __shared__ u32 cnt;
    const u64 limit = min(total, ctl->solver_c);  // nothing at or above the first solver is admitted
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const u64 c = (u64)blockIdx.x * RES_CTA + threadIdx.x;
    bool win = false;
    if (c < limit) {
        u32 s = slot[c];
        if (s != LTL_NONE) win = ld_rank(table + s) == gbase + c;
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, win);
    if ((threadIdx.x & 31) == 0) {
        flagw[c >> 5] = b;
        if (b) atomicAdd(&cnt, __popc(b));
    }
    __syncthreads();
    if (threadIdx.x == 0) blocksum[blockIdx.x] = cnt;
}

// exclusive scan of the block sums (single CTA) -> blockoff, ctl->total
__global__ void __launch_bounds__(1024) k_scan(const u32* __restrict__ blocksum, u32 nb, u64* __restrict__ blockoff,
                                               Ctl* ctl) {
    __shared__ u64 wsum[32];
    __shared__ u64 carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (u32 base = 0; base < nb; base += 1024) {
        const u32 idx = base + threadIdx.x;
        const u64 v = idx < nb ? blocksum[idx] : 0;
        u64 x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            u64 w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                u64 y = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const u64 before = carry + (warp ? wsum[warp - 1] : 0) + (x - v);
        if (idx < nb) blockoff[idx] = before;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) ctl->total = carry;
}

// winners (in rank order) -> records at entry n_base + dest; the first winner beyond the budget marks OOM
__global__ void __launch_bounds__(RES_CTA) k_emit(const u32* __restrict__ flagw, const u64* __restrict__ blockoff,
                                                  const Piece* __restrict__ pieces, int n_pieces, u64 total, i64 n_base,
                                                  u64 cap_left, unsigned char* __restrict__ rec_op,
                                                  int* __restrict__ rec_lhs, int* __restrict__ rec_rhs,
                                                  u32* __restrict__ dest_out, Ctl* ctl) {
    __shared__ u32 wcnt[32];
    const u64 limit = min(total, ctl->solver_c);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u64 c = (u64)blockIdx.x * RES_CTA + threadIdx.x;
    const u32 fw = flagw[c >> 5];
    if (lane == 0) wcnt[warp] = __popc(fw);
    __syncthreads();
    if (c < total) dest_out[c] = LTL_NONE;  // every candidate gets a verdict: the tile-shaped phase B reads it
    if (!((fw >> lane) & 1u) || c >= limit) return;
    u64 dest = blockoff[blockIdx.x] + __popc(fw & ((1u << lane) - 1u));
    for (int w = 0; w < warp; w++) dest += wcnt[w];
    if (dest > cap_left) return;
    if (dest == cap_left) {
        ctl->oom_c = c;
        return;
    }
    dest_out[c] = (u32)dest;
    int lo = 0, hi = n_pieces - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if ((u64)pieces[mid].cbase <= c) lo = mid;
        else hi = mid - 1;
    }
    const Piece pc = pieces[lo];
    i64 i, j;
    piece_unrank(pc, c, &i, &j);
    const i64 e = n_base + (i64)dest;
    rec_op[e] = (unsigned char)pc.op;
    rec_lhs[e] = (int)i;
    rec_rhs[e] = (int)j;
}

// Small passes (cost levels of a few thousand candidates are bound by launch latency, not by work): ONE CTA does what
// k_finalize + k_resolve + k_scan + k_emit do for big passes -- complete the row-split candidates, decide the winners
// (lowest rank per key), compact them in rank order and write their records -- 1024 candidates per round with a running
// offset.  It also zeroes the partial sums it consumed, so the next small pass needs no memset.
#define LTL_SMALL_SCREEN 8192
#define LTL_SMALL_ADMIT 8192  // (one CTA takes ~1.5 us per 1024 candidates: at 20 K candidates -- config 5, cost level 6 --
                              // it cost 32 us where the four full-width kernels need 18)
template <bool MUELLER>
__global__ void __launch_bounds__(RES_CTA) k_admit_small(const __grid_constant__ ScreenParams p, u64 total, int finalize,
                                                         i64 n_base, u64 cap_left, unsigned char* __restrict__ rec_op,
                                                         int* __restrict__ rec_lhs, int* __restrict__ rec_rhs,
                                                         u32* __restrict__ dest_out) {
    __shared__ u32 wcnt[32];
    __shared__ u64 carry_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (finalize) {
        for (u64 c = threadIdx.x; c < total; c += RES_CTA) {
            finish_candidate<MUELLER>(p, c, p.acc[3 * c], p.acc[3 * c + 1], (u32)p.acc[3 * c + 2]);
            p.acc[3 * c] = 0;
            p.acc[3 * c + 1] = 0;
            p.acc[3 * c + 2] = 0;
        }
        __threadfence();
    }
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const u64 limit = min(total, *((volatile u64*)&p.ctl->solver_c));  // nothing at or above the first solver is admitted
    for (u64 base = 0; base < total; base += RES_CTA) {
        const u64 c = base + threadIdx.x;
        bool win = false;
        if (c < limit) {
            const u32 s = p.slot[c];
            if (s != LTL_NONE) win = ld_rank(p.table + s) == p.gbase + c;
        }
        const unsigned b = __ballot_sync(0xFFFFFFFFu, win);
        if (lane == 0) wcnt[warp] = __popc(b);
        __syncthreads();
        u64 dest = carry_s + __popc(b & ((1u << lane) - 1u));
        u32 block_total = 0;
        for (int w = 0; w < 32; w++) {
            const u32 v = wcnt[w];
            if (w < warp) dest += v;
            block_total += v;
        }
        if (c < total) dest_out[c] = LTL_NONE;  // every candidate gets a verdict: the tile-shaped phase B reads it
        if (win) {
            if (dest == cap_left) p.ctl->oom_c = c;  // the first winner beyond the budget marks OOM
            else if (dest < cap_left) {
                dest_out[c] = (u32)dest;
                int lo = 0, hi = p.n_pieces - 1;
                while (lo < hi) {
                    int mid = (lo + hi + 1) >> 1;
                    if ((u64)p.pieces[mid].cbase <= c) lo = mid;
                    else hi = mid - 1;
                }
                const Piece pc = p.pieces[lo];
                i64 i, j;
                piece_unrank(pc, c, &i, &j);
                const i64 e = n_base + (i64)dest;
                rec_op[e] = (unsigned char)pc.op;
                rec_lhs[e] = (int)i;
                rec_rhs[e] = (int)j;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) carry_s += block_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) p.ctl->total = carry_s;
}

// ---- phase-B order.  Phase B re-derives every winner from its record, in entry order = rank order: for a
// piece op(i, j) that is "for each left operand i: all right operands j".  When the right bucket is larger than L2 every
// i streams it from DRAM again (ncu, config 2: 19.7 GB read to write 21 GB, L2 hit rate 12.7 %).  The entry order is
// fixed, the PROCESSING order is not: the winners of (i, block of right operands) are one run of consecutive entries,
// found from the winner flags of the admission pass, and phase B walks the runs block by block -- "for each block of j:
// all i (of every connective over that bucket)" -- so a block is read from DRAM once and from L2 afterwards.
//
// winners with chunk-local rank < c (flag words + per-1024 offsets of k_resolve / k_scan)
__device__ __forceinline__ u64 winners_before(const u32* __restrict__ flagw, const u64* __restrict__ blockoff, u64 c, u64 total,
                                              u64 all_winners) {
    if (c >= total) return all_winners;
    u64 d = blockoff[c >> 10];
    const u64 w0 = (c >> 10) << 5, w1 = c >> 5;
    for (u64 w = w0; w < w1; w++) d += __popc(flagw[w]);
    return d + __popc(flagw[w1] & ((1u << (c & 31)) - 1u));
}

__global__ void k_mat_plan(const PlanFam* __restrict__ fams, int n_fams, i64 n_threads, const Piece* __restrict__ pieces,
                           const u32* __restrict__ flagw, const u64* __restrict__ blockoff, const Ctl* __restrict__ ctl,
                           u64 total, i64 n_base, u64 count, u32* __restrict__ seg_g0, u32* __restrict__ seg_cnt) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_threads) return;
    int lo = 0, hi = n_fams - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (fams[mid].t_base <= t) lo = mid;
        else hi = mid - 1;
    }
    const PlanFam f = fams[lo];
    const Piece pc = pieces[f.piece];
    u64 c_lo, c_hi;
    i64 pos;
    if (f.n_jb == 0) {
        c_lo = (u64)pc.cbase;
        c_hi = (u64)(pc.cbase + pc.count);
        pos = f.pos_base;
    } else {
        const i64 local = t - f.t_base;
        const i64 jb = local / f.n_i, ii = local - jb * f.n_i;
        const i64 nj = pc.j1 - pc.j0;
        const i64 b_lo = (pc.j0 / f.block + jb) * f.block;
        const i64 jlo = max(pc.j0, b_lo), jhi = min(pc.j1, b_lo + f.block);
        c_lo = (u64)(pc.cbase + ii * nj + (jlo - pc.j0));
        c_hi = (u64)(pc.cbase + ii * nj + (jhi - pc.j0));
        pos = f.pos_base + jb * f.stride + f.off + ii;
    }
    const u64 all_winners = ctl->total;
    const u64 a = min(winners_before(flagw, blockoff, c_lo, total, all_winners), count);
    const u64 b = min(winners_before(flagw, blockoff, c_hi, total, all_winners), count);
    // a group belongs to the run that holds its first new entry
    const i64 g_base = n_base >> 5;
    const i64 ga = a == 0 ? g_base : ((n_base + (i64)a + 31) >> 5);
    const i64 gb = b == 0 ? g_base : ((n_base + (i64)b + 31) >> 5);
    seg_g0[pos] = (u32)(ga - g_base);
    seg_cnt[pos] = (u32)(gb - ga);
}

// exclusive scan of up to 2^16 run lengths (single CTA): off[0 .. n], off[n] = total groups
__global__ void __launch_bounds__(1024) k_plan_scan(const u32* __restrict__ cnt, int n, u32* __restrict__ off) {
    __shared__ u32 wsum[32];
    __shared__ u32 carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < n; base += 1024) {
        const int idx = base + threadIdx.x;
        const u32 v = idx < n ? cnt[idx] : 0u;
        u32 x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            u32 w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 y = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const u32 before = carry + (warp ? wsum[warp - 1] : 0u) + (x - v);
        if (idx < n) off[idx] = before;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[n] = carry;
}

// entry e <- proposition words resident on the device (ltl_traces): optionally negated inside the mask, optionally
// packed two rows per word (half-width store).  n = stored words per entry, R = rows (one word each when pair).
__global__ void k_import_dev(const u64* __restrict__ src, const u64* __restrict__ masks, int negated, int pair, i64 R,
                             u64* __restrict__ cms, i64 e, i64 n) {
    const i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    auto val = [&](i64 i) -> u64 { return negated ? ~src[i] & masks[i] : src[i]; };
    u64 word;
    if (pair) word = (val(2 * k) & 0xFFFFFFFF00000000ull) | (2 * k + 1 < R ? val(2 * k + 1) >> 32 : 0ull);
    else word = val(k);
    cms[cm_index(e, n, k)] = word;
}

// masks of the half-width store from one-word row masks
__global__ void k_pack_pairs(const u64* __restrict__ rows, i64 R, u64* __restrict__ out, i64 n) {
    const i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    out[k] = (rows[2 * k] & 0xFFFFFFFF00000000ull) | (2 * k + 1 < R ? rows[2 * k + 1] >> 32 : 0ull);
}

__global__ void k_import(const u64* __restrict__ stage, u64* __restrict__ cms, i64 e, i64 n) {
    i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) cms[cm_index(e, n, k)] = stage[k];
}

// out[(e - first) * n + k] for entries [first, first + count)
__global__ void k_export(const u64* __restrict__ cms, i64 first, i64 count, i64 n, u64* __restrict__ out) {
    const i64 g0 = first >> 5;
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const i64 lane = t & 31;
    const i64 gk = t >> 5;
    const i64 g = gk / n, k = gk - g * n;
    const i64 e = (g0 + g) * 32 + lane;
    if (e >= first && e < first + count) out[(size_t)(e - first) * n + k] = cms[cm_index(e, n, k)];
}

// debug invariant of the reference (bitsem.py:46-61, LTLLEARN_DEBUG_MASKS): no characteristic bit outside the validity mask
__global__ void k_check_masks(const u64* __restrict__ cms, const u64* __restrict__ masks, i64 first, i64 count, i64 n,
                              u64* __restrict__ bad) {
    const i64 g0 = first >> 5;
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const i64 lane = t & 31;
    const i64 gk = t >> 5;
    const i64 g = gk / n, k = gk - g * n;
    const i64 e = (g0 + g) * 32 + lane;
    if (e >= first && e < first + count && (cms[cm_index(e, n, k)] & ~masks[k])) atomicAdd(bad, 1ull);
}

__global__ void k_found_to_acc(const Ctl* ctl, u64* acc) {
    acc[0] = ctl->found;
    acc[1] = acc[2] = 0;
}
__global__ void k_acc_to_found(Ctl* ctl, u64* acc) {
    ctl->found = acc[0] ? 1ull : 0ull;
    acc[0] = 0;
}

__global__ void k_set_record(unsigned char* rec_op, int* rec_lhs, int* rec_rhs, i64 e, int op, int lhs, int rhs) {
    rec_op[e] = (unsigned char)op;
    rec_lhs[e] = lhs;
    rec_rhs[e] = rhs;
}

__global__ void k_rehash(const Slot* __restrict__ old, u64 old_cap, Slot* __restrict__ fresh, u64 fresh_mask) {
    u64 s = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= old_cap) return;
    const Key128 k = ld_key(old + s);
    if (k.hi == ~0ull) return;
    u64 d = table_find_or_claim(fresh, fresh_mask, k.hi, k.lo);
    fresh[d].rank = old[s].rank;
}

// after a solve / OOM cut: keys filed by candidates at or above the cut are not members
__global__ void k_purge(Slot* table, u64 cap, u64 gcut) {
    u64 s = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= cap) return;
    if (table[s].hi == ~0ull) return;
    u64 r = table[s].rank;
    if (r != LTL_RANK_NONE && r >= gcut) table[s].rank = LTL_RANK_NONE;
}

// ---- multi-GPU stages (sharded.py): the owner of a fingerprint files (hi, lo, global rank) tuples received
// from every rank, then says which tuple owns its key
__global__ void k_file_insert(const u64* __restrict__ tuples, u64 count, Slot* table, u64 mask, u64 gbase,
                              u32* __restrict__ slot_out) {
    u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const u64 hi = tuples[3 * t], lo = tuples[3 * t + 1], rank = tuples[3 * t + 2];
    const u64 s = table_find_or_claim(table, mask, hi, lo);
    const u64 old = atomicMin(&table[s].rank, rank);
    slot_out[t] = old < gbase ? LTL_NONE : (u32)s;
}

__global__ void k_file_verdict(const u64* __restrict__ tuples, const u32* __restrict__ slot, u64 count,
                               const Slot* __restrict__ table, unsigned char* __restrict__ win, Ctl* ctl) {
    u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    bool w = false;
    if (t < count) {
        const u32 s = slot[t];
        w = s != LTL_NONE && ld_rank(table + s) == tuples[3 * t + 2];
        win[t] = w ? 1 : 0;
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, w);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(&ctl->total, (u64)__popc(b));
}

// ---- candidate-range shards: routing of (fingerprint, rank) tuples to their hash owners, on the device ----------------
#define LTL_MAX_WORLD 64

// pass 1 of a stable counting sort by owner: hist[d * nb + block] = tuples of this 1024-tuple block owned by rank d
__global__ void __launch_bounds__(1024) k_route_count(const u64* __restrict__ fp, u64 count, int world, u32* __restrict__ hist, u32 nb) {
    __shared__ u32 cnt[LTL_MAX_WORLD];
    if (threadIdx.x < LTL_MAX_WORLD) cnt[threadIdx.x] = 0;
    __syncthreads();
    const u64 t = (u64)blockIdx.x * 1024 + threadIdx.x;
    const int d = t < count ? fp_owner(fp[2 * t], fp[2 * t + 1], world) : LTL_MAX_WORLD;
    const unsigned m = __match_any_sync(0xFFFFFFFFu, d);
    if (d < LTL_MAX_WORLD && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&cnt[d], (u32)__popc(m));
    __syncthreads();
    if ((int)threadIdx.x < world) hist[(size_t)threadIdx.x * nb + blockIdx.x] = cnt[threadIdx.x];
}

// pass 2: tuple t goes to off[owner * nb + block] + (tuples of the same owner before it in its block): grouped by owner,
// in rank order inside a group
__global__ void __launch_bounds__(1024) k_route_scatter(const u64* __restrict__ fp, u64 count, int world, u64 rank_base,
                                                        const u32* __restrict__ off, u32 nb, u64* __restrict__ send) {
    __shared__ u32 wc[32][LTL_MAX_WORLD];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < 32 * LTL_MAX_WORLD; k += 1024) (&wc[0][0])[k] = 0;
    __syncthreads();
    const u64 t = (u64)blockIdx.x * 1024 + threadIdx.x;
    u64 hi = 0, lo = 0;
    int d = LTL_MAX_WORLD;
    if (t < count) {
        hi = fp[2 * t];
        lo = fp[2 * t + 1];
        d = fp_owner(hi, lo, world);
    }
    const unsigned m = __match_any_sync(0xFFFFFFFFu, d);
    const u32 in_warp = (u32)__popc(m & ((1u << lane) - 1u));
    if (d < LTL_MAX_WORLD && lane == __ffs(m) - 1) wc[warp][d] = (u32)__popc(m);
    __syncthreads();
    if ((int)threadIdx.x < world) {  // exclusive prefix over the warps, per owner
        u32 run = 0;
        for (int w = 0; w < 32; w++) {
            const u32 v = wc[w][threadIdx.x];
            wc[w][threadIdx.x] = run;
            run += v;
        }
    }
    __syncthreads();
    if (d < LTL_MAX_WORLD) {
        const size_t pos = (size_t)off[(size_t)d * nb + blockIdx.x] + wc[warp][d] + in_warp;
        send[3 * pos] = hi;
        send[3 * pos + 1] = lo;
        send[3 * pos + 2] = rank_base + t;
    }
}

// verdicts come back in the order the tuples were sent: set the winner bit of the tuple's candidate
__global__ void k_win_flags(const u64* __restrict__ tuples, const unsigned char* __restrict__ win, u64 count, u64 rank_base,
                            u32* __restrict__ flagw) {
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count || !win[t]) return;
    const u64 c = tuples[3 * t + 2] - rank_base;
    atomicOr(flagw + (c >> 5), 1u << (c & 31));
}

__global__ void __launch_bounds__(RES_CTA) k_flag_count(const u32* __restrict__ flagw, u64 count, u32* __restrict__ blocksum) {
    __shared__ u32 cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const u64 c = (u64)blockIdx.x * RES_CTA + threadIdx.x;
    if ((threadIdx.x & 31) == 0 && c < count) {
        const u32 b = flagw[c >> 5];
        if (b) atomicAdd(&cnt, (u32)__popc(b));
    }
    __syncthreads();
    if (threadIdx.x == 0) blocksum[blockIdx.x] = cnt;
}

// the winners' level ranks, ascending
__global__ void __launch_bounds__(RES_CTA) k_emit_ranks(const u32* __restrict__ flagw, const u64* __restrict__ blockoff, u64 count,
                                                        i64 level_lo, i64* __restrict__ out) {
    __shared__ u32 wcnt[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u64 c = (u64)blockIdx.x * RES_CTA + threadIdx.x;
    const u32 fw = c < count ? flagw[c >> 5] : 0u;
    if (lane == 0) wcnt[warp] = __popc(fw);
    __syncthreads();
    if (!((fw >> lane) & 1u)) return;
    u64 dest = blockoff[blockIdx.x] + __popc(fw & ((1u << lane) - 1u));
    for (int w = 0; w < warp; w++) dest += wcnt[w];
    out[dest] = level_lo + (i64)c;
}

// the records of a formula: every entry reachable from `root` through (lhs, rhs), each once, root first -- one launch and
// one copy instead of one device round trip per node (reference cache.py:197-213 walks get_record node by node)
#define LTL_SUBTREE_MAX 4096
__global__ void k_subtree(const unsigned char* __restrict__ rec_op, const int* __restrict__ rec_lhs, const int* __restrict__ rec_rhs,
                          i64 root, i64 n_entries, int cap, int* __restrict__ out /* [cap][4]: entry, op, lhs, rhs */, int* __restrict__ n_out) {
    int n = 0, head = 0;
    if (root >= 0 && root < n_entries && cap > 0) {
        out[0] = (int)root;
        n = 1;
    }
    while (head < n) {  // breadth first over the list itself
        const int e = out[4 * head];
        const int op = rec_op[e], lhs = rec_lhs[e], rhs = rec_rhs[e];
        out[4 * head + 1] = op;
        out[4 * head + 2] = lhs;
        out[4 * head + 3] = rhs;
        head++;
        if (op == OP_IDENT) continue;  // an atom: lhs is the proposition
        const bool unary = op == OP_NOT || op == OP_NEXT || op == OP_FINALLY || op == OP_GLOBALLY;
        for (int k = 0; k < (unary ? 1 : 2); k++) {
            const int child = k == 0 ? lhs : rhs;
            if (child < 0 || child >= n_entries) continue;  // dangling: the caller reports it
            bool seen = false;
            for (int q = 0; q < n; q++) seen |= out[4 * q] == child;
            if (!seen && n < cap) out[4 * n++] = child;
            else if (!seen) {
                *n_out = -1;  // more nodes than the buffer holds
                return;
            }
        }
    }
    *n_out = n;
}

// level ranks -> records
__global__ void k_decode(const i64* __restrict__ ranks, u64 count, const Piece* __restrict__ pieces, int n_pieces,
                         unsigned char* __restrict__ op, int* __restrict__ lhs, int* __restrict__ rhs) {
    u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const u64 c = (u64)ranks[t];
    int lo = 0, hi = n_pieces - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if ((u64)pieces[mid].cbase <= c) lo = mid;
        else hi = mid - 1;
    }
    const Piece pc = pieces[lo];
    i64 i, j;
    piece_unrank(pc, c, &i, &j);
    op[t] = (unsigned char)pc.op;
    lhs[t] = (int)i;
    rhs[t] = (int)j;
}

// ------------------------------------------------------------------------------------------------
// driver API (virtual memory management) through the runtime's entry-point lookup: no link-time libcuda

struct DriverApi {
    bool tried = false, ok = false;
    CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
};

static DriverApi& drv() {
    static DriverApi d;
    if (d.tried) return d;
    d.tried = true;
    if (getenv("LTL_NO_VMM")) return d;
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
            !*fn)
            ok = false;
    };
    get("cuMemAddressReserve", (void**)&d.MemAddressReserve);
    get("cuMemAddressFree", (void**)&d.MemAddressFree);
    get("cuMemCreate", (void**)&d.MemCreate);
    get("cuMemRelease", (void**)&d.MemRelease);
    get("cuMemMap", (void**)&d.MemMap);
    get("cuMemUnmap", (void**)&d.MemUnmap);
    get("cuMemSetAccess", (void**)&d.MemSetAccess);
    get("cuMemGetAllocationGranularity", (void**)&d.MemGetAllocationGranularity);
    cudaGetLastError();
    d.ok = ok;
    return d;
}

// A device buffer that grows in place: a reserved virtual range, physical memory mapped on demand
// (180 GB of HBM is filled without ever copying the store).  Falls back to malloc + copy without VMM.
static bool pool_enabled() {
    static int on = -1;
    if (on < 0) on = getenv("LTL_NO_POOL") ? 0 : 1;
    return on == 1;
}

struct GrowBuf {
    char* base = nullptr;
    size_t reserved = 0, mapped = 0, gran = 0;
    bool vmm = false;
    int device = 0;
    std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> parts;

    int init(int dev, size_t max_bytes) {
        device = dev;
        DriverApi& d = drv();
        if (d.ok) {
            CUmemAllocationProp prop;
            memset(&prop, 0, sizeof(prop));
            prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            prop.location.id = dev;
            if (d.MemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && gran) {
                size_t want = ((max_bytes + gran - 1) / gran) * gran;
                if (want < gran) want = gran;
                CUdeviceptr p = 0;
                if (d.MemAddressReserve(&p, want, 0, 0, 0) == CUDA_SUCCESS) {
                    base = (char*)p;
                    reserved = want;
                    vmm = true;
                    return 0;
                }
            }
        }
        vmm = false;
        reserved = max_bytes;
        return 0;
    }

    // 0 ok, -1 device out of memory / failure
    int ensure(size_t bytes, cudaStream_t stream) {
        if (bytes <= mapped) return 0;
        if (bytes > reserved) return -1;
        if (vmm) {
            DriverApi& d = drv();
            size_t step = std::max(mapped / 4, (size_t)(64u << 20));
            size_t target = std::max(bytes, std::min(reserved, mapped + step));
            target = std::min(reserved, ((target + gran - 1) / gran) * gran);
            for (int attempt = 0; attempt < 2; attempt++) {
                size_t add = target - mapped;
                CUmemAllocationProp prop;
                memset(&prop, 0, sizeof(prop));
                prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
                prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
                prop.location.id = device;
                CUmemGenericAllocationHandle hnd;
                if (d.MemCreate(&hnd, add, &prop, 0) == CUDA_SUCCESS) {
                    if (d.MemMap((CUdeviceptr)(base + mapped), add, 0, hnd, 0) != CUDA_SUCCESS) {
                        d.MemRelease(hnd);
                        return -1;
                    }
                    CUmemAccessDesc acc;
                    memset(&acc, 0, sizeof(acc));
                    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
                    acc.location.id = device;
                    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
                    if (d.MemSetAccess((CUdeviceptr)(base + mapped), add, &acc, 1) != CUDA_SUCCESS) {
                        d.MemUnmap((CUdeviceptr)(base + mapped), add);
                        d.MemRelease(hnd);
                        return -1;
                    }
                    parts.push_back({hnd, add});
                    mapped = target;
                    return 0;
                }
                // retry with exactly what is needed
                target = std::min(reserved, ((bytes + gran - 1) / gran) * gran);
                if (target <= mapped) return -1;
            }
            return -1;
        }
        size_t target = std::min(reserved, std::max(bytes, std::max(mapped * 2, (size_t)(1u << 20))));
        char* fresh = nullptr;
        if (cudaMalloc(&fresh, target) != cudaSuccess) {
            cudaGetLastError();
            target = bytes;
            if (cudaMalloc(&fresh, target) != cudaSuccess) {
                cudaGetLastError();
                return -1;
            }
        }
        if (base) {
            cudaMemcpyAsync(fresh, base, mapped, cudaMemcpyDeviceToDevice, stream);
            cudaStreamSynchronize(stream);
            cudaFree(base);
        }
        base = fresh;
        mapped = target;
        return 0;
    }

    void release() {
        if (vmm) {
            DriverApi& d = drv();
            size_t off = 0;
            for (auto& pr : parts) {
                d.MemUnmap((CUdeviceptr)(base + off), pr.second);
                d.MemRelease(pr.first);
                off += pr.second;
            }
            parts.clear();
            if (base) d.MemAddressFree((CUdeviceptr)base, reserved);
        } else if (base) {
            cudaFree(base);
        }
        base = nullptr;
        mapped = reserved = 0;
    }
};

// ------------------------------------------------------------------------------------------------
// the core object

struct KStat {
    u64 launches = 0, units = 0;
    double ms = 0, bytes = 0;
};

struct PendingEvent {
    int cls;
    cudaEvent_t a, b;
};

// An admitted range whose matrices are still to be written.  While d_dest still holds the verdicts of the pass
// that admitted it (`tiled`), phase B runs tile-shaped over the same pieces as phase A; otherwise from records.
struct PendingMat {
    u64 n_base = 0, count = 0;
    bool tiled = false;
    bool small_rows = false;  // multi-word rows, a small pass: one lane per (entry, row) (k_materialize_small_rows)
    int n_seg = 0;  // > 0: the phase-B order of this range is in the core's plan buffers
    std::vector<Piece> pieces;
    i64 total = 0, tiles = 0;
};

// a unit of enumeration before chunking
struct Unit {
    int kind, op, seg;
    i64 i0, i1, j0, j1;
};

static thread_local std::string g_create_error;

// Every device / pinned resource of a core.  Released arenas are pooled per process and handed to the next
// core on the same device (a learner creates one core per search, divide-and-conquer many): mapping,
// unmapping and (de)allocating tens of GB costs far more than a search and varies wildly between runs, so in
// steady state a search performs no memory-management call at all.
struct Arena {
    int device = -1;
    cudaStream_t stream = nullptr;
    u64* d_masks = nullptr;
    i64 masks_cap = 0;
    Deposit* d_deps = nullptr;
    int deps_cap = 0;
    GrowBuf cms, rec_op, rec_lhs, rec_rhs;
    Slot* table = nullptr;
    u64 table_cap = 0;
    i64 scratch_cap = 0;
    u32* d_slot = nullptr;
    u32* d_dest = nullptr;  // per candidate of the last admission pass: index among the winners / NONE
    u32* d_flagw = nullptr;
    u32* d_blocksum = nullptr;
    u64* d_blockoff = nullptr;
    u64* d_acc = nullptr;  // per-candidate partial sums (s0, s1, errors): row-split passes, row shards
    i64 acc_cap = 0;
    u64* d_fp = nullptr;
    i64 fp_cap = 0;
    Piece* d_pieces = nullptr;
    Piece* h_pieces = nullptr;
    int pieces_cap = 0;
    Ctl* d_ctl = nullptr;
    Ctl* h_ctl = nullptr;
    u64* d_stage = nullptr;
    u64* h_stage = nullptr;  // pinned
    i64 stage_cap = 0;
    cudaEvent_t sub_ev[2] = {nullptr, nullptr};
    u64* h_solver = nullptr;  // pinned: solver rank as of the end of each of the last two phase-A launches
    LevelsState* d_lv = nullptr;  // device-resident cost levels (levels.cuh): search state on the device ...
    LevelsState* h_lv = nullptr;  // ... and its pinned host copy
    std::vector<cudaEvent_t> event_pool;

    void destroy_all() {
        if (device < 0) return;
        cudaSetDevice(device);
        for (auto e : event_pool) cudaEventDestroy(e);
        event_pool.clear();
        if (sub_ev[0]) cudaEventDestroy(sub_ev[0]);
        if (sub_ev[1]) cudaEventDestroy(sub_ev[1]);
        cudaFreeHost(h_solver);
        cudaFree(d_lv);
        cudaFreeHost(h_lv);
        cms.release();
        rec_op.release();
        rec_lhs.release();
        rec_rhs.release();
        cudaFree(table);
        cudaFree(d_masks);
        cudaFree(d_deps);
        cudaFree(d_slot);
        cudaFree(d_dest);
        cudaFree(d_flagw);
        cudaFree(d_blocksum);
        cudaFree(d_blockoff);
        cudaFree(d_acc);
        cudaFree(d_fp);
        cudaFree(d_pieces);
        cudaFree(d_ctl);
        cudaFree(d_stage);
        cudaFreeHost(h_pieces);
        cudaFreeHost(h_ctl);
        cudaFreeHost(h_stage);
        if (stream) cudaStreamDestroy(stream);
        cudaGetLastError();
        *this = Arena();
    }
};

static std::mutex g_pool_mutex;
static std::vector<Arena>& g_pool() {
    static std::vector<Arena> pool;
    return pool;
}

static bool pool_take(int device, Arena& out) {
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    auto& pool = g_pool();
    int best = -1;
    for (int k = 0; k < (int)pool.size(); k++)
        if (pool[k].device == device && (best < 0 || pool[k].cms.mapped > pool[best].cms.mapped)) best = k;
    if (best < 0) return false;
    out = pool[best];
    pool.erase(pool.begin() + best);
    return true;
}

static void pool_give(Arena& a) {
    if (pool_enabled() && a.device >= 0) {
        std::lock_guard<std::mutex> lock(g_pool_mutex);
        if (g_pool().size() < 16) {
            g_pool().push_back(a);
            a = Arena();
            return;
        }
    }
    a.destroy_all();
}

static size_t pool_trim() {  // give every pooled page back to the driver
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    size_t freed = 0;
    for (auto& a : g_pool()) {
        freed += a.cms.mapped + a.table_cap * sizeof(Slot);
        a.destroy_all();
    }
    g_pool().clear();
    return freed;
}

struct ltl_core : Arena {
    // Half-width store (`pair`, variant NH32: every trace has at most 32 positions): two rows share one stored word
    // (row 2v high half, row 2v + 1 low half), so R / n / n_pos below count STORED words -- R = ceil(R_api / 2),
    // n_pos = positive high-half rows, n_pos_lo = positive low-half rows -- while the C ABI keeps uint64[R_api].
    int R = 0, W = 0, n_pos = 0, err_max = 0, variant = 0, fkp_bits = 0, mask_k = 0;
    int R_api = 0, n_pos_lo = 0;
    bool pair = false;
    i64 n = 0, n_api = 0;
    u64 budget = 0, entry_bytes = 0;
    u64 cap_entries = 0;  // admissions allowed: min(logical budget, what the device can hold)
    int n_dep = 0;
    u64 keys_upper = 0;
    i64 chunk_cap = 1 << 28;  // candidates per ordered-admission pass (normally a whole cost level)
    double deadline_at = 0;   // steady-clock seconds after which run_level stops between passes (0: none)
    i64 sub_tiles = 1 << 16;  // warp tiles per phase-A launch: little work is issued after a solver shows up (2^15: +2.4 %
                              // step time on the bench workload from the drained tails between launches; >= 2^16: equal)
    u64 n_entries = 0, offered = 0, admitted = 0, duplicates = 0;
    u64 h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic of this handle
    double exchange_ms = 0;  // host wall time inside the row-shard exchange callback
    double grow_ms = 0, sync_ms = 0, plan_ms = 0;  // host wall time: store growth, waiting for the device, planning
    int sm_count = 148;
    int max_split = 4096, force_split = 0;
    bool fuse_unary = true;
    // row shard (ltl_core_set_row_shard): this core holds rows of every matrix starting at word 64 * blk_base of the
    // whole matrix; partial sums are summed across the shards by `exchange` before candidates are completed
    u64 pending_purge = ~0ull;  // global rank cut of a solve / OOM whose table sweep has not run yet
    u32 blk_base = 0;
    ltl_exchange_fn exchange = nullptr;
    void* exchange_ctx = nullptr;
    bool fuse_not = true;  // phase B of a level also screens NOT(new entry) for the next level (k_materialize_not)
    bool gate_store = true;  // ... and writes the matrices only if the pass it is issued behind found no solver (run_chunk)
    i64 fuse_not_min = 32768;
    u64 gated_skips = 0;  // conditional phase-B launches that found the gate closed (statistics)  // ... when it writes at least this many entries: the fused kernel folds all rows of an
                               // entry in one lane (no row split), which is slow on a launch that cannot fill the SMs
    int tiled_materialize = -1;  // phase B over phase A's tiles instead of per record: 1 always, 0 never, -1 by size
    bool device_oom = false;      // an S_OOM came from the device, not from the logical budget
    bool store_results = true;    // false: admitted entries get records and fingerprints but no matrix
    bool debug_masks = false;     // check every matrix written against the validity masks (reference LTLLEARN_DEBUG_MASKS)
    u64* d_dbg = nullptr;
    int* d_subtree = nullptr;
    u32 *d_route_hist = nullptr, *d_route_off = nullptr;  // candidate-range shards: owner histogram / offsets of stage_route
    size_t route_cap = 0;
    cudaEvent_t part_ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int exchange_parts = 4;       // row shards: parts of a pass whose exchange overlaps the evaluation of the next part
    u64 exchange_calls = 0;
    int table_shard = 0, table_shards = 1;  // row shards: this core files only the keys it owns (fp_owner), see set_table_shard
    bool order_mat = true;        // phase B walks big right-operand buckets block by block (k_mat_plan)
    i64 order_min = 1 << 16;      // ... for passes that admit at least this many entries
    i64 order_block_bytes = 16 << 20;
    u32 *d_plan_g0 = nullptr, *d_plan_cnt = nullptr, *d_plan_off = nullptr;
    PlanFam* d_plan_fams = nullptr;
    int plan_cap = 0, plan_fams_cap = 0;
    bool plan_in_use = false;
    bool small_screen = true;     // small passes over one-word rows: the compact phase-A kernel (k_screen_small)
    bool small_admit = true;      // passes of <= LTL_SMALL_ADMIT candidates: one bookkeeping kernel instead of four
    bool device_levels = true;    // run_search: the first (small) cost levels in one launch, planned on the device (levels.cuh)
    int levels_ctas = LTL_LV_MAX_CLUSTER;  // CTAs of that launch's cluster
    i64 levels_max_work = (i64)1 << 18;    // candidate-rows per level up to which a level stays in that launch (8 SMs: beyond,
                                           // the host-driven path with the whole GPU behind it is faster -- measured)
    bool acc_dirty = true;        // the partial-sum arrays may hold something other than zeros
    u64 unstored_from = ~0ull;    // first entry index without a stored matrix
    bool profile = false;
    KStat stats[LTL_K_COUNT];
    std::vector<PendingEvent> pending;
    u64* fp_ext = nullptr;  // MODE_FP_ONLY output override (device pointer owned by the caller)
    std::vector<PendingMat> pending_mat;  // admitted ranges whose matrices are not yet written
    std::string err;

    int fail(int code, const std::string& msg) {
        err = msg;
        return code;
    }
    int cuda_fail(cudaError_t e, const char* what) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        cudaGetLastError();
        return LTL_ERR_CUDA;
    }
};

#define CK(call)                                        \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return h->cuda_fail(e_, #call); \
    } while (0)

static cudaEvent_t get_event(ltl_core* h) {
    if (!h->event_pool.empty()) {
        cudaEvent_t e = h->event_pool.back();
        h->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ScopedTimer {
    ltl_core* h;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    ScopedTimer(ltl_core* h_, int cls_, u64 units, double bytes) : h(h_), cls(cls_) {
        h->stats[cls].launches++;
        h->stats[cls].units += units;
        h->stats[cls].bytes += bytes;
        if (h->profile) {
            a = get_event(h);
            b = get_event(h);
            cudaEventRecord(a, h->stream);
        }
    }
    ~ScopedTimer() {
        if (a) {
            cudaEventRecord(b, h->stream);
            h->pending.push_back({cls, a, b});
        }
    }
};

static void drain_events(ltl_core* h) {  // stream must be idle
    for (auto& pe : h->pending) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, pe.a, pe.b) == cudaSuccess) h->stats[pe.cls].ms += ms;
        h->event_pool.push_back(pe.a);
        h->event_pool.push_back(pe.b);
    }
    h->pending.clear();
    cudaGetLastError();
}

static int ensure_table(ltl_core* h, u64 need_keys) {
    if (h->exchange && h->table_shards > 1)  // a shard of the table: the keys this core owns (+ 25 % for an uneven split)
        need_keys = need_keys / (u64)h->table_shards + need_keys / (4 * (u64)h->table_shards) + 1024;
    u64 want = 1u << 16;
    while (want < need_keys * 2) want <<= 1;
    if (want <= h->table_cap) return LTL_OK;
    if (want > (1ull << 31)) return h->fail(LTL_ERR_DEVICE_OOM, "uniqueness table would exceed 2^31 slots");
    Slot* fresh = nullptr;
    if (cudaMalloc(&fresh, want * sizeof(Slot)) != cudaSuccess) {
        cudaGetLastError();
        return h->fail(LTL_ERR_DEVICE_OOM, "device memory exhausted growing the uniqueness table");
    }
    CK(cudaMemsetAsync(fresh, 0xFF, want * sizeof(Slot), h->stream));
    if (h->table) {
        {
            ScopedTimer t(h, LTL_K_REHASH, h->table_cap, (double)h->table_cap * sizeof(Slot));
            k_rehash<<<(unsigned)((h->table_cap + 255) / 256), 256, 0, h->stream>>>(h->table, h->table_cap, fresh, want - 1);
        }
        CK(cudaStreamSynchronize(h->stream));
        drain_events(h);
        cudaFree(h->table);
    }
    h->table = fresh;
    h->table_cap = want;
    return LTL_OK;
}

static int flush_materialize(ltl_core* h, const ScreenParams* sp = nullptr, int fuse_kind = 0, i64 not_cbase = 0, i64 not_i0 = 0,
                             const u64* store_gate = nullptr);
static int check_masks(ltl_core* h, u64 first, u64 count);

static int ensure_scratch(ltl_core* h, i64 total) {
    if (total <= h->scratch_cap) return LTL_OK;
    for (auto& pm : h->pending_mat)
        if (pm.tiled) {  // the verdict array is about to be reallocated
            int rcf = flush_materialize(h);
            if (rcf) return rcf;
            break;
        }
    i64 cap = std::max<i64>(total, std::min<i64>(h->chunk_cap, std::max<i64>(h->scratch_cap * 4, 1 << 16)));
    cap = ((cap + RES_CTA - 1) / RES_CTA) * RES_CTA;
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(h->d_slot);
    cudaFree(h->d_dest);
    cudaFree(h->d_flagw);
    cudaFree(h->d_blocksum);
    cudaFree(h->d_blockoff);
    h->d_slot = h->d_dest = nullptr;
    h->d_flagw = h->d_blocksum = nullptr;
    h->d_blockoff = nullptr;
    h->scratch_cap = 0;
    CK(cudaMalloc(&h->d_slot, (size_t)cap * 4));
    CK(cudaMalloc(&h->d_dest, (size_t)cap * 4));
    CK(cudaMalloc(&h->d_flagw, (size_t)(cap / 32) * 4 + 64));  // (+ zeroed slack: the flags are exchanged in units of 3 words)
    CK(cudaMemsetAsync((char*)h->d_flagw + (size_t)(cap / 32) * 4, 0, 64, h->stream));
    CK(cudaMalloc(&h->d_blocksum, (size_t)(cap / RES_CTA) * 4));
    CK(cudaMalloc(&h->d_blockoff, (size_t)(cap / RES_CTA) * 8));
    h->scratch_cap = cap;
    return LTL_OK;
}

static int ensure_acc(ltl_core* h, i64 total) {
    if (total <= h->acc_cap) return LTL_OK;
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(h->d_acc);
    h->d_acc = nullptr;
    h->acc_cap = 0;
    i64 cap = std::max<i64>(total, 1 << 12);
    CK(cudaMalloc(&h->d_acc, (size_t)cap * 24));
    h->acc_cap = cap;
    h->acc_dirty = true;
    return LTL_OK;
}

static int ensure_pieces(ltl_core* h, int n) {
    if (n <= h->pieces_cap) return LTL_OK;
    int cap = std::max(n, std::max(64, h->pieces_cap * 2));
    CK(cudaStreamSynchronize(h->stream));
    cudaFree(h->d_pieces);
    cudaFreeHost(h->h_pieces);
    h->d_pieces = h->h_pieces = nullptr;
    h->pieces_cap = 0;
    CK(cudaMalloc(&h->d_pieces, sizeof(Piece) * cap));
    CK(cudaMallocHost(&h->h_pieces, sizeof(Piece) * cap));
    h->pieces_cap = cap;
    return LTL_OK;
}

struct HostTimer {
    double* acc;
    std::chrono::steady_clock::time_point t0;
    explicit HostTimer(double* a) : acc(a), t0(std::chrono::steady_clock::now()) {}
    ~HostTimer() { *acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};

static int ensure_entries(ltl_core* h, u64 entries) {  // matrices + records for `entries` entries
    HostTimer ht(&h->grow_ms);
    const u64 groups = (entries + 31) / 32;
    for (int attempt = 0; attempt < 2; attempt++) {
        if (!(h->cms.ensure((size_t)groups * 32 * (size_t)h->n * 8, h->stream) || h->rec_op.ensure((size_t)groups * 32, h->stream) ||
              h->rec_lhs.ensure((size_t)groups * 32 * 4, h->stream) || h->rec_rhs.ensure((size_t)groups * 32 * 4, h->stream)))
            return LTL_OK;
        cudaGetLastError();
        if (attempt == 0 && pool_trim() == 0) break;
    }
    return h->fail(LTL_ERR_DEVICE_OOM, "device memory exhausted growing the entry store");
}

static int ensure_records(ltl_core* h, u64 entries) {
    const u64 groups = (entries + 31) / 32;
    if (h->rec_op.ensure((size_t)groups * 32, h->stream) || h->rec_lhs.ensure((size_t)groups * 32 * 4, h->stream) ||
        h->rec_rhs.ensure((size_t)groups * 32 * 4, h->stream)) {
        cudaGetLastError();
        return h->fail(LTL_ERR_DEVICE_OOM, "device memory exhausted growing the record store");
    }
    return LTL_OK;
}

// ------------------------------------------------------------------------------------------------
// chunk planning

static inline bool is_binary(int op) { return op == OP_AND || op == OP_OR || op == OP_UNTIL; }

static void push_piece(ltl_core* h, std::vector<Piece>& pieces, i64& total, i64& tiles, const Unit& u, i64 i0, i64 i1,
                       i64 j0, i64 j1, int kind, bool ext = false) {
    Piece p;
    memset(&p, 0, sizeof(p));
    p.op = u.op;
    p.kind = kind;
    p.seg = u.seg;
    p.i0 = i0;
    p.i1 = i1;
    p.j0 = j0;
    p.j1 = j1;
    p.swap = 0;
    p.ti = 1;
    p.owns_tiles = 1;
    i64 lane_lo, lane_hi, rows;
    if (kind == PIECE_UNARY) {
        p.count = i1 - i0;
        lane_lo = i0;
        lane_hi = i1;
        rows = 1;
    } else if (kind == PIECE_RECT) {
        p.count = (i1 - i0) * (j1 - j0);
        p.swap = (i1 - i0) > (j1 - j0) ? 1 : 0;
        lane_lo = p.swap ? i0 : j0;
        lane_hi = p.swap ? i1 : j1;
        rows = p.swap ? (j1 - j0) : (i1 - i0);
    } else {
        p.count = (i64)tri_before((u64)(i1 - i0), (u64)(j1 - 1 - i0));
        lane_lo = i0 + 1;
        lane_hi = j1;
        rows = i1 - i0;
    }
    if (kind != PIECE_UNARY && h->W == 1 && (h->variant == VAR_MUELLER || h->variant == VAR_NH)) p.ti = 4;
    p.lane_g0 = lane_lo >> 5;
    p.tiles_lane = ((lane_hi - 1) >> 5) - p.lane_g0 + 1;
    const i64 row_tiles = (rows + p.ti - 1) / p.ti;
    p.tiles_row = row_tiles;
    p.cbase = total;
    p.tile_base = tiles;
    total += p.count;
    if (ext) {  // evaluated by phase B of the entries it ranges over (fused NOT): ranks, but no tiles
        p.ext = 1;
        p.owns_tiles = 0;
        pieces.push_back(p);
        return;
    }
    // fuse with an earlier unary piece over the same operand range (same chunk): it evaluates this connective too
    if (kind == PIECE_UNARY && h->W == 1 && (h->variant == VAR_MUELLER || h->variant == VAR_NH) && h->fuse_unary && p.op != OP_IDENT) {
        for (auto& q : pieces) {
            if (q.kind != PIECE_UNARY || q.i0 != i0 || q.i1 != i1 || q.nfuse == 0 || q.nfuse >= 4) continue;
            if (((q.fops >> (4 * (q.nfuse - 1))) & 15) >= p.op) continue;  // keep nibbles in ascending opcode order
            // only rank-adjacent pieces fuse (NEXT, FINALLY, GLOBALLY follow one another in the enumeration
            // order; NOT is followed by the binary connectives): the launch order stays the rank order
            if (q.fcbase[q.nfuse - 1] + q.count != p.cbase) continue;
            q.fops |= p.op << (4 * q.nfuse);
            q.fcbase[q.nfuse] = p.cbase;
            q.nfuse++;
            p.nfuse = 0;  // sibling: owns no tiles
            p.owns_tiles = 0;
            pieces.push_back(p);
            return;
        }
        p.nfuse = 1;
        p.fops = p.op;
        p.fcbase[0] = p.cbase;
    }
    tiles += row_tiles * p.tiles_lane;
    pieces.push_back(p);
}

// Expand caller segments into rectangular / triangular / unary units (reference _speedups.pyx:364-368:
// for row i the columns start at max(b0, i + 1) when tri).
static int expand_segments(ltl_core* h, const ltl_segment* segs, int n_segs, std::vector<Unit>& units) {
    const i64 ne = (i64)h->n_entries;
    for (int s = 0; s < n_segs; s++) {
        const ltl_segment& g = segs[s];
        const bool unary = g.op == OP_NOT || g.op == OP_NEXT || g.op == OP_FINALLY || g.op == OP_GLOBALLY;
        if (!unary && !is_binary(g.op)) return h->fail(LTL_ERR_ARG, "segment: unknown opcode");
        if (g.a0 < 0 || g.a1 > ne || g.a0 > g.a1) return h->fail(LTL_ERR_ARG, "segment: left range outside the store");
        if ((u64)g.a1 > h->unstored_from || (!unary && g.b1 > 0 && (u64)g.b1 > h->unstored_from))
            return h->fail(LTL_ERR_ARG, "segment: operand matrices were not stored (store_results was off)");
        if (unary) {
            if (g.a1 > g.a0) units.push_back({PIECE_UNARY, g.op, s, g.a0, g.a1, -1, -1});
            continue;
        }
        if (g.b0 < 0 || g.b1 > ne || g.b0 > g.b1) return h->fail(LTL_ERR_ARG, "segment: right range outside the store");
        if (g.a1 == g.a0 || g.b1 == g.b0) continue;
        if (!g.tri) {
            units.push_back({PIECE_RECT, g.op, s, g.a0, g.a1, g.b0, g.b1});
            continue;
        }
        const i64 rect_end = std::min(g.a1, g.b0);  // rows i < b0 see the whole right range
        if (g.a0 < rect_end) units.push_back({PIECE_RECT, g.op, s, g.a0, rect_end, g.b0, g.b1});
        const i64 t0 = std::max(g.a0, g.b0), t1 = std::min(g.a1, g.b1 - 1);  // row b1-1 has no column left
        if (t0 < t1) units.push_back({PIECE_TRI, g.op, s, t0, t1, -1, g.b1});
    }
    return LTL_OK;
}

// ------------------------------------------------------------------------------------------------
// one chunk

// lowest chunk-local rank a warp tile of a piece can hold (mirrors the early-exit test in k_screen)
static i64 tile_min_rank(const Piece& pc, i64 t) {
    const bool lane_major = pc.kind == PIECE_RECT && pc.swap;
    const i64 minor = lane_major ? pc.tiles_row : pc.tiles_lane;
    const i64 hi_ = t / minor, lo_ = t - hi_ * minor;
    const i64 rt = lane_major ? lo_ : hi_;
    const i64 lfirst = (pc.lane_g0 + (lane_major ? hi_ : lo_)) * 32;
    if (pc.kind == PIECE_UNARY) return (i64)piece_rank(pc, std::max(lfirst, pc.i0), -1);
    if (pc.kind == PIECE_RECT && pc.swap) return (i64)piece_rank(pc, std::max(lfirst, pc.i0), pc.j0 + rt * pc.ti);
    const i64 row0 = pc.i0 + rt * pc.ti;
    if (pc.kind == PIECE_RECT) return (i64)piece_rank(pc, row0, std::max(lfirst, pc.j0));
    return (i64)piece_rank(pc, row0, std::max(lfirst, row0 + 1));
}

struct ChunkOut {
    int status = LTL_S_DONE;
    u64 cut_c = ~0ull;  // chunk-local rank of the solving / overflowing candidate
    u64 admitted = 0;
};

static void choose_split(ltl_core* h, i64 tiles, int* nsplit, int* rows_per_split) {
    int ns = 1;  // (tiles == 0: a pass whose only candidates are the NOTs that phase B screens -- found by scripts/soak.py)
    const i64 target = (i64)h->sm_count * 16 * 4;  // warps wanted: 4 waves, so uneven tiles still balance
    if (h->force_split > 0) ns = h->force_split;
    else if (tiles > 0 && tiles < target && h->R >= 2 * LTL_SPLIT_ROWS) ns = (int)std::min<i64>((target + tiles - 1) / tiles, h->max_split);
    const int max_ns = (h->R + LTL_SPLIT_ROWS - 1) / LTL_SPLIT_ROWS;
    ns = std::max(1, std::min(ns, max_ns));
    int rps = (h->R + ns - 1) / ns;
    rps = ((rps + LTL_SPLIT_ROWS - 1) / LTL_SPLIT_ROWS) * LTL_SPLIT_ROWS;
    *rows_per_split = rps;
    *nsplit = (h->R + rps - 1) / rps;
}

static double screen_bytes(ltl_core* h, const std::vector<Piece>& pieces) {
    double b = 0;
    const double B = 8.0 * (double)h->n;
    for (auto& p : pieces)
        if (!p.ext) b += (double)p.count * ((p.kind == PIECE_UNARY ? 1.0 : 2.0) * B + 16.0);
    return b;
}

// fused_not >= 0: index of the piece (ext) whose candidates NOT(entry) are screened by phase B of the pending entries,
// which this pass therefore issues itself, right before its own phase A launches
static int apply_purge(ltl_core* h) {
    if (h->pending_purge == ~0ull) return LTL_OK;
    {
        ScopedTimer t(h, LTL_K_PURGE, h->table_cap, (double)h->table_cap * sizeof(Slot));
        k_purge<<<(unsigned)((h->table_cap + 255) / 256), 256, 0, h->stream>>>(h->table, h->table_cap, h->pending_purge);
    }
    CK(cudaGetLastError());
    h->pending_purge = ~0ull;
    return LTL_OK;
}

// Phase-B order of the range just admitted (see k_mat_plan): runs of consecutive new entries, by (right-operand bucket,
// block of it, connective, left operand).  Needs the winner flags of the admission pass that is still in the scratch
// arrays, so it is issued right behind it.  Returns the number of runs (0: keep the entry order).
static int plan_materialize(ltl_core* h, const std::vector<Piece>& pieces, i64 total, u64 n_base, u64 count, int* n_seg_out) {
    *n_seg_out = 0;
    if (!h->order_mat || h->plan_in_use || (i64)count < h->order_min) return LTL_OK;
    const i64 block = std::max<i64>(32, (h->order_block_bytes / (8 * h->n)) & ~(i64)31);
    std::vector<PlanFam> fams;
    fams.reserve(pieces.size());
    // pieces over the same right bucket share its blocks: their runs interleave block by block
    struct Group {
        i64 j0, j1, n_jb, sum_i, pos_base;
    };
    std::vector<Group> groups;
    std::vector<int> fam_group;
    bool any_split = false;
    for (size_t k = 0; k < pieces.size(); k++) {
        const Piece& pc = pieces[k];
        if (pc.count <= 0) continue;
        PlanFam f;
        memset(&f, 0, sizeof(f));
        f.piece = (int)k;
        f.block = block;
        const i64 nj = pc.j1 - pc.j0;
        const bool split = pc.kind == PIECE_RECT && nj >= 2 * block && pc.i1 - pc.i0 >= 2;
        int gi = -1;
        if (split) {
            f.n_i = pc.i1 - pc.i0;
            f.n_jb = (int)((pc.j1 - 1) / block - pc.j0 / block + 1);
            for (size_t g = 0; g < groups.size(); g++)
                if (groups[g].j0 == pc.j0 && groups[g].j1 == pc.j1) gi = (int)g;
            if (gi < 0) {
                groups.push_back({pc.j0, pc.j1, f.n_jb, 0, 0});
                gi = (int)groups.size() - 1;
            }
            f.off = groups[(size_t)gi].sum_i;
            groups[(size_t)gi].sum_i += f.n_i;
            any_split = true;
        }
        fams.push_back(f);
        fam_group.push_back(gi);
    }
    if (!any_split) return LTL_OK;
    // positions: runs in rank order, except that the pieces of a group are laid out together where its first piece stands
    i64 pos = 0, threads = 0;
    std::vector<char> placed(groups.size(), 0);
    for (size_t k = 0; k < fams.size(); k++) {
        PlanFam& f = fams[k];
        f.t_base = threads;
        const int gi = fam_group[k];
        if (gi < 0) {
            f.pos_base = pos++;
            threads += 1;
            continue;
        }
        Group& g = groups[(size_t)gi];
        if (!placed[(size_t)gi]) {
            placed[(size_t)gi] = 1;
            g.pos_base = pos;
            pos += g.n_jb * g.sum_i;
        }
        f.pos_base = g.pos_base;
        f.stride = g.sum_i;
        threads += (i64)f.n_jb * f.n_i;
    }
    if (pos > (1 << 16) || pos < 2) return LTL_OK;
    const int n_seg = (int)pos;
    if (n_seg + 1 > h->plan_cap) {
        CK(cudaStreamSynchronize(h->stream));
        cudaFree(h->d_plan_g0);
        cudaFree(h->d_plan_cnt);
        cudaFree(h->d_plan_off);
        h->d_plan_g0 = h->d_plan_cnt = h->d_plan_off = nullptr;
        h->plan_cap = 0;
        const int cap = std::max(n_seg + 1, 4096);
        CK(cudaMalloc(&h->d_plan_g0, (size_t)cap * 4));
        CK(cudaMalloc(&h->d_plan_cnt, (size_t)cap * 4));
        CK(cudaMalloc(&h->d_plan_off, (size_t)cap * 4));
        h->plan_cap = cap;
    }
    if ((int)fams.size() > h->plan_fams_cap) {
        CK(cudaStreamSynchronize(h->stream));
        cudaFree(h->d_plan_fams);
        h->d_plan_fams = nullptr;
        h->plan_fams_cap = 0;
        const int cap = std::max((int)fams.size(), 256);
        CK(cudaMalloc(&h->d_plan_fams, sizeof(PlanFam) * (size_t)cap));
        h->plan_fams_cap = cap;
    }
    CK(cudaMemcpyAsync(h->d_plan_fams, fams.data(), sizeof(PlanFam) * fams.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));  // `fams` is pageable and goes out of scope (the caller syncs here anyway)
    h->h2d_bytes += sizeof(PlanFam) * fams.size();
    {
        ScopedTimer t(h, LTL_K_MISC, (u64)threads, (double)threads * 64.0);
        k_mat_plan<<<(unsigned)((threads + 255) / 256), 256, 0, h->stream>>>(h->d_plan_fams, (int)fams.size(), threads, h->d_pieces,
                                                                            h->d_flagw, h->d_blockoff, h->d_ctl, (u64)total,
                                                                            (i64)n_base, count, h->d_plan_g0, h->d_plan_cnt);
        k_plan_scan<<<1, 1024, 0, h->stream>>>(h->d_plan_cnt, n_seg, h->d_plan_off);
        h->stats[LTL_K_MISC].launches += 1;  // (two kernels under one timer)
    }
    CK(cudaGetLastError());
    h->plan_in_use = true;
    *n_seg_out = n_seg;
    return LTL_OK;
}

static int run_chunk(ltl_core* h, std::vector<Piece>& pieces, i64 total, i64 tiles, int mode, bool check_solve,
                     bool materialize, ChunkOut* out, int fused_not = -1) {
    int rc;
    if (total <= 0) return LTL_OK;
    if ((rc = apply_purge(h))) return rc;
    if (mode == MODE_INSERT) {
        bool tiled_pending = false;
        for (auto& pm : h->pending_mat) tiled_pending |= pm.tiled;
        if (tiled_pending && (rc = flush_materialize(h))) return rc;  // this pass overwrites the verdicts they need
        if ((rc = ensure_table(h, h->keys_upper + (u64)total))) return rc;
        if ((rc = ensure_scratch(h, total))) return rc;
        const u64 room = h->cap_entries > h->n_entries ? h->cap_entries - h->n_entries : 0;
        if ((rc = ensure_records(h, h->n_entries + std::min<u64>((u64)total, room) + 1))) return rc;
    }
    if ((rc = ensure_pieces(h, (int)pieces.size()))) return rc;
    memcpy(h->h_pieces, pieces.data(), sizeof(Piece) * pieces.size());
    CK(cudaMemcpyAsync(h->d_pieces, h->h_pieces, sizeof(Piece) * pieces.size(), cudaMemcpyHostToDevice, h->stream));
    h->h2d_bytes += sizeof(Piece) * pieces.size();
    if (mode == MODE_INSERT) {  // solver_c = oom_c = none; `total` is assigned by the scan, nothing else is read
        CK(cudaMemsetAsync(h->d_ctl, 0xFF, sizeof(Ctl), h->stream));
    } else {
        CK(cudaMemsetAsync(h->d_ctl, 0xFF, 2 * sizeof(u64), h->stream));
        CK(cudaMemsetAsync((char*)h->d_ctl + 2 * sizeof(u64), 0, sizeof(Ctl) - 2 * sizeof(u64), h->stream));
    }
    // (row shards with a sharded table exchange the winner flags between resolve and scan: the four-kernel path)
    const bool small = mode == MODE_INSERT && h->small_admit && total <= LTL_SMALL_ADMIT && !(h->exchange && h->table_shards > 1);

    ScreenParams p;
    memset(&p, 0, sizeof(p));
    p.cms = (const u64*)h->cms.base;
    p.masks = h->d_masks;
    p.pieces = h->d_pieces;
    p.n_pieces = (int)pieces.size();
    p.R = h->R;
    p.W = h->W;
    p.n_pos = h->n_pos;
    p.n_pos_lo = h->n_pos_lo;
    p.pair = h->pair ? 1 : 0;
    p.err_max = h->err_max;
    p.n = h->n;
    p.total_tiles = tiles;
    choose_split(h, tiles, &p.nsplit, &p.rows_per_split);
    // small passes over one-word rows go through the compact kernel: blocks of 64 rows per thread
    // (rows of 2 / 4 / 8 / 16 words tile the 64-word hash blocks: k_screen_small_rows, NH only)
    const bool small_rows_w = (h->W == 2 || h->W == 4 || h->W == 8 || h->W == 16) && h->variant == VAR_NH;
    const bool small_screen = h->small_screen && (h->W == 1 || small_rows_w) && !h->pair && mode != MODE_REWRITE &&
                              total <= LTL_SMALL_SCREEN && (i64)total * h->n <= ((i64)1 << (h->W == 1 ? 24 : 22)) && h->force_split == 0 &&
                              !h->exchange && h->R <= 65535 * LTL_SPLIT_ROWS;
    if (small_screen) {
        p.rows_per_split = LTL_SPLIT_ROWS;
        p.nsplit = (h->R + LTL_SPLIT_ROWS - 1) / LTL_SPLIT_ROWS;
    }
    p.variant = h->variant;
    p.mask_k = h->mask_k;
    p.n_dep = h->n_dep;
    p.deps = h->d_deps;
    p.mode = mode;
    p.check_solve = check_solve ? 1 : 0;
    p.table = h->table;
    p.table_mask = h->table_cap ? h->table_cap - 1 : 0;
    p.gbase = h->offered;
    p.slot = h->d_slot;
    p.fp_out = mode == MODE_FP_ONLY ? (h->fp_ext ? h->fp_ext : h->d_fp) : nullptr;
    p.ctl = h->d_ctl;
    p.blk_base = h->blk_base;
    p.defer = h->exchange ? 1 : 0;
    p.owner_world = h->exchange ? h->table_shards : 1;
    p.owner_rank = h->table_shard;
    const bool acc_path = p.nsplit > 1 || p.defer || (small_screen && h->W > 1);  // (the multi-word small kernel always sums blocks)
    if (acc_path) {
        if ((rc = ensure_acc(h, total))) return rc;
        p.acc = h->d_acc;
        // (the small-pass bookkeeping kernel leaves the sums it consumed zeroed: nothing to clear between small passes)
        const size_t clear = (size_t)(small ? std::max<i64>(total, std::min<i64>(h->acc_cap, LTL_SMALL_ADMIT)) : total);
        // (a row shard without row split stores every candidate's sums exactly once: nothing to clear)
        const bool stored = p.defer && p.nsplit == 1;
        if (!stored && (!small || h->acc_dirty)) {
            CK(cudaMemsetAsync(h->d_acc, 0, clear * 24, h->stream));
        }
        h->acc_dirty = stored ? true : !small;
    }
    u64 issued_units = 0;       // what the phase-A launches of this pass were booked with (statistics)
    double issued_bytes = 0;
    const bool mueller = h->variant == VAR_MUELLER || h->variant == VAR_NH;  // hashed variants: two 64-bit sums
    const int screen_kind = h->variant == VAR_MUELLER ? KIND_MUELLER : h->variant == VAR_NH ? KIND_NH : KIND_BITS;
    // Phase B of the newest level with this level's NOT fused in.  The pieces in front of the first one that reads those
    // matrices -- the level's AND / OR candidates: binary connectives pair cheaper operands -- do not need them, so when the
    // solver rank of a tile is final once the tile has run (no partial sums to combine afterwards) the launch goes out
    // BEHIND their tiles and stores only if they found no solver: the search that solves there (BASELINE config 2: 2.56 M
    // entries, 21 GB) never writes the largest level it admitted.  Tiles behind the gate are launched after it in stream
    // order: either the matrices are there by then, or a solver below them is known and they return at once.
    const bool gated = fused_not >= 0 && h->gate_store && !p.defer && !acc_path && !small_screen;
    const size_t n_pending_before = h->pending_mat.size();
    i64 gate_tile = tiles;  // first tile of the first piece that reads a pending entry
    if (gated) {
        const i64 pend0 = (i64)h->pending_mat.front().n_base;
        for (size_t k = 0; k < pieces.size(); k++) {
            const Piece& pc = pieces[k];
            if (pc.ext || !pc.owns_tiles || (int)k == fused_not) continue;
            if (pc.i1 > pend0 || (pc.kind != PIECE_UNARY && pc.j1 > pend0)) {
                gate_tile = pc.tile_base;
                break;
            }
        }
    }
    bool gate_issued = false;
    auto issue_gate = [&]() -> int {
        const Piece& fp = pieces[(size_t)fused_not];
        gate_issued = true;
        CK(cudaMemcpyAsync(&h->d_ctl->gate, &h->d_ctl->solver_c, sizeof(u64), cudaMemcpyDeviceToDevice, h->stream));
        return flush_materialize(h, &p, screen_kind, fp.cbase, fp.i0, &h->d_ctl->gate);
    };
    if (fused_not >= 0 && !gated) {
        const Piece& fp = pieces[(size_t)fused_not];
        if ((rc = flush_materialize(h, &p, screen_kind, fp.cbase, fp.i0))) return rc;
    }
    if (gated)  // room for the matrices is mapped before anything is filed: running out of device memory ends the level cleanly
        for (auto& pm : h->pending_mat)
            if ((rc = ensure_entries(h, pm.n_base + pm.count))) return rc;
    if (small_screen) {
        ScopedTimer t(h, LTL_K_SCREEN, (u64)total, screen_bytes(h, pieces));
        issued_units = (u64)total;
        issued_bytes = screen_bytes(h, pieces);
        if (h->W == 1) ltl_launch_screen_small(p, screen_kind, (unsigned long long)total, h->stream);
        else if (h->W == 2) ltl_launch_screen_small_w2(p, (unsigned long long)total, h->stream);
        else if (h->W == 4) ltl_launch_screen_small_w4(p, (unsigned long long)total, h->stream);
        else if (h->W == 8) ltl_launch_screen_small_w8(p, (unsigned long long)total, h->stream);
        else ltl_launch_screen_small_w16(p, (unsigned long long)total, h->stream);
        CK(cudaGetLastError());
    } else if (p.defer) {
        // Row shards: every shard adds its partial sums, then all of them complete identical candidates.  The pass is cut
        // at piece boundaries into up to `exchange_parts` parts (contiguous ranges of tiles AND of ranks); all parts are
        // launched at once, and while part k + 1 is still being evaluated the sums of part k -- complete as soon as its
        // launch has ended -- are already being all-reduced: the exchange overlaps phase A instead of following it.
        struct Part {
            i64 t0, t1, c0, c1;
        };
        std::vector<Part> parts;
        {
            const i64 want = std::max<i64>(1, std::min<i64>(h->exchange_parts, 8));
            i64 t_start = 0, c_start = 0;
            for (size_t k = 1; k < pieces.size(); k++) {
                if (!pieces[k].owns_tiles || pieces[k].ext) continue;  // siblings stay with the piece that evaluates them
                const i64 goal = tiles * (i64)(parts.size() + 1) / want;
                if ((i64)parts.size() + 1 < want && pieces[k].tile_base >= goal && pieces[k].tile_base > t_start) {
                    parts.push_back({t_start, pieces[k].tile_base, c_start, pieces[k].cbase});
                    t_start = pieces[k].tile_base;
                    c_start = pieces[k].cbase;
                }
            }
            parts.push_back({t_start, tiles, c_start, total});
        }
        const double bytes_all = screen_bytes(h, pieces);
        for (size_t k = 0; k < parts.size(); k++) {
            const Part& pt = parts[k];
            if (pt.t1 > pt.t0) {
                const double frac = tiles > 0 ? (double)(pt.t1 - pt.t0) / (double)tiles : 0.0;
                ScopedTimer t(h, LTL_K_SCREEN, (u64)((double)total * frac), bytes_all * frac);
                issued_units += (u64)((double)total * frac);
                issued_bytes += bytes_all * frac;
                dim3 grid((unsigned)(((pt.t1 - pt.t0) * p.nsplit + LTL_WARPS_PER_CTA - 1) / LTL_WARPS_PER_CTA), 1);
                ScreenParams q = p;
                q.tile_offset = pt.t0;
                q.total_tiles = pt.t1;
                (h->pair ? ltl_launch_screen_w1p : SCREEN_FN[h->W])(q, screen_kind, grid, h->stream);
            }
            if (!h->part_ev[k]) CK(cudaEventCreateWithFlags(&h->part_ev[k], cudaEventDisableTiming));
            CK(cudaEventRecord(h->part_ev[k], h->stream));
        }
        CK(cudaGetLastError());
        for (size_t k = 0; k < parts.size(); k++) {
            const Part& pt = parts[k];
            {
                HostTimer ht(&h->sync_ms);
                CK(cudaEventSynchronize(h->part_ev[k]));
            }
            if (pt.c1 <= pt.c0) continue;
            HostTimer ht(&h->exchange_ms);
            if (h->exchange(h->exchange_ctx, h->d_acc + 3 * pt.c0, (int64_t)(pt.c1 - pt.c0)))
                return h->fail(LTL_ERR_CUDA, "row-shard exchange failed");
            h->exchange_calls++;
        }
    } else {
        // Phase A goes out in launches of sub_tiles warp tiles, in enumeration order, with no host wait in
        // between (two in flight); after each one the solver rank is copied to pinned memory, and once a solver is
        // known no launch is issued whose first tile lies above it.
        {
            // (fingerprint-only passes that look for a solver -- the sharded evaluation stage -- stop early too)
            const bool whole = acc_path || mode == MODE_LOOKUP || (mode == MODE_FP_ONLY && !check_solve);
            const i64 per = whole ? tiles : std::max<i64>(h->sub_tiles, LTL_WARPS_PER_CTA);
            const double bytes_all = screen_bytes(h, pieces);
            issued_units = 0;
            issued_bytes = 0;
            u64 known_solver = ~0ull;
            int k = 0;
            for (i64 t0 = 0, t1 = 0; t0 < tiles; t0 = t1, k++) {
                if (gated && !gate_issued && t0 >= gate_tile && (rc = issue_gate())) return rc;
                t1 = std::min(tiles, t0 + per);
                if (gated && !gate_issued && t1 > gate_tile) t1 = gate_tile;  // (t0 < gate_tile here)
                if (per < tiles) {
                    if (k >= 2) {
                        HostTimer ht(&h->sync_ms);
                        CK(cudaEventSynchronize(h->sub_ev[k & 1]));
                        known_solver = std::min(known_solver, h->h_solver[k & 1]);
                    }
                    if (known_solver != ~0ull && check_solve) {
                        // first tile of this launch: its piece and the lowest rank it can hold
                        size_t pi = 0;
                        for (size_t q = 0; q < pieces.size(); q++)
                            if (pieces[q].owns_tiles && pieces[q].tile_base <= t0) pi = q;
                        if ((u64)tile_min_rank(pieces[pi], t0 - pieces[pi].tile_base) > known_solver) break;
                    }
                }
                p.tile_offset = t0;
                const double frac = (double)(t1 - t0) / (double)tiles;
                ScopedTimer t(h, LTL_K_SCREEN, (u64)((double)total * frac), bytes_all * frac);
                issued_units += (u64)((double)total * frac);
                issued_bytes += bytes_all * frac;
                dim3 grid((unsigned)(((t1 - t0) * p.nsplit + LTL_WARPS_PER_CTA - 1) / LTL_WARPS_PER_CTA), 1);
                ScreenParams q = p;
                q.total_tiles = t1;
                (h->pair ? ltl_launch_screen_w1p : SCREEN_FN[h->W])(q, screen_kind, grid, h->stream);
                if (per < tiles) {
                    CK(cudaMemcpyAsync(h->h_solver + (k & 1), &h->d_ctl->solver_c, sizeof(u64), cudaMemcpyDeviceToHost, h->stream));
                    CK(cudaEventRecord(h->sub_ev[k & 1], h->stream));
                }
            }
        }
        CK(cudaGetLastError());
    }
    if (gated && !gate_issued && (rc = issue_gate())) return rc;  // (no tile behind the gate, or phase A stopped at a solver)
    if (acc_path && !small) {
        ScopedTimer t(h, LTL_K_FINALIZE, (u64)total, (double)total * 36.0);
        if (mueller) k_finalize<true><<<(unsigned)((total + 255) / 256), 256, 0, h->stream>>>(p, (u64)total);
        else k_finalize<false><<<(unsigned)((total + 255) / 256), 256, 0, h->stream>>>(p, (u64)total);
        CK(cudaGetLastError());
    }
    if (mode == MODE_LOOKUP && p.owner_world > 1) {  // only the key's owner knows: OR over the shards
        k_found_to_acc<<<1, 1, 0, h->stream>>>(h->d_ctl, h->d_acc);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
        if (h->exchange(h->exchange_ctx, h->d_acc, 1)) return h->fail(LTL_ERR_CUDA, "row-shard exchange failed");
        k_acc_to_found<<<1, 1, 0, h->stream>>>(h->d_ctl, h->d_acc);
        CK(cudaGetLastError());
    }
    if (mode != MODE_INSERT) {
        CK(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->d2h_bytes += sizeof(Ctl);
        drain_events(h);
        return LTL_OK;
    }

    // ---- ordered admission.  The resolve limit min(total, solver rank) is read from ctl on the device, so
    // phase A and the three bookkeeping kernels run back to back with one host round trip per chunk.
    const u64 room = h->cap_entries > h->n_entries ? h->cap_entries - h->n_entries : 0;
    if (small) {
        {
            ScopedTimer t(h, LTL_K_RESOLVE, (u64)total, (double)total * (acc_path ? 72.0 : 36.0));
            if (mueller)
                k_admit_small<true><<<1, RES_CTA, 0, h->stream>>>(p, (u64)total, acc_path ? 1 : 0, (i64)h->n_entries, room,
                                                                  (unsigned char*)h->rec_op.base, (int*)h->rec_lhs.base,
                                                                  (int*)h->rec_rhs.base, h->d_dest);
            else
                k_admit_small<false><<<1, RES_CTA, 0, h->stream>>>(p, (u64)total, acc_path ? 1 : 0, (i64)h->n_entries, room,
                                                                   (unsigned char*)h->rec_op.base, (int*)h->rec_lhs.base,
                                                                   (int*)h->rec_rhs.base, h->d_dest);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
        {
            HostTimer ht(&h->sync_ms);
            CK(cudaStreamSynchronize(h->stream));
        }
        h->d2h_bytes += sizeof(Ctl);
    } else {
        const unsigned nb = (unsigned)((total + RES_CTA - 1) / RES_CTA);
        {
            ScopedTimer t(h, LTL_K_RESOLVE, (u64)total, (double)total * 36.0);
            k_resolve<<<nb, RES_CTA, 0, h->stream>>>(h->d_slot, h->table, h->offered, (u64)total, h->d_ctl, h->d_flagw,
                                                      h->d_blocksum);
        }
        if (p.owner_world > 1) {
            // every shard decided the keys it owns: the winner flags (one bit per candidate, set by one shard at most)
            // are OR-ed over the shards -- as a wrapping sum of disjoint bits, 3 words per exchange unit
            const i64 words = (i64)nb * (RES_CTA / 64);
            {
                HostTimer ht(&h->sync_ms);
                CK(cudaStreamSynchronize(h->stream));
            }
            {
                HostTimer ht(&h->exchange_ms);
                if (h->exchange(h->exchange_ctx, h->d_flagw, (words + 2) / 3)) return h->fail(LTL_ERR_CUDA, "row-shard exchange failed");
                h->exchange_calls++;
            }
            ScopedTimer t(h, LTL_K_RESOLVE, (u64)total, (double)total * 0.125);
            k_flag_count<<<nb, RES_CTA, 0, h->stream>>>(h->d_flagw, (u64)nb * RES_CTA, h->d_blocksum);
        }
        {
            ScopedTimer t(h, LTL_K_SCAN, nb, (double)nb * 12.0);
            k_scan<<<1, 1024, 0, h->stream>>>(h->d_blocksum, nb, h->d_blockoff, h->d_ctl);
        }
        {
            ScopedTimer t(h, LTL_K_EMIT, (u64)total, (double)total * 0.125);
            k_emit<<<nb, RES_CTA, 0, h->stream>>>(h->d_flagw, h->d_blockoff, h->d_pieces, (int)pieces.size(), (u64)total,
                                                   (i64)h->n_entries, room, (unsigned char*)h->rec_op.base,
                                                   (int*)h->rec_lhs.base, (int*)h->rec_rhs.base, h->d_dest, h->d_ctl);
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
        {
            HostTimer ht(&h->sync_ms);
            CK(cudaStreamSynchronize(h->stream));
        }
        h->d2h_bytes += sizeof(Ctl);
    }
    const u64 solver_c = h->h_ctl->solver_c;
    const u64 winners = h->h_ctl->total;
    const u64 oom_c = h->h_ctl->oom_c;
    drain_events(h);
    if (gated) {
        if (h->h_ctl->gate == ~0ull) {  // the gate was open: the pending ranges are written
            if (h->debug_masks)
                for (size_t k = 0; k < n_pending_before; k++)
                    if ((rc = check_masks(h, h->pending_mat[k].n_base, h->pending_mat[k].count))) {
                        h->pending_mat.clear();
                        return rc;
                    }
            h->pending_mat.erase(h->pending_mat.begin(), h->pending_mat.begin() + (std::ptrdiff_t)n_pending_before);
        } else {  // closed: they stay pending (read-backs write them), and the launch is booked as the NOT pass it was
            for (size_t k = 0; k < n_pending_before; k++) {
                h->pending_mat[k].n_seg = 0;  // (the plan arrays may be reused by then: entry order)
                h->stats[LTL_K_MATERIALIZE].bytes -= (double)h->pending_mat[k].count * 25.0;
            }
            h->gated_skips++;
        }
    }
    const bool oom = winners > room;
    const u64 count = oom ? room : winners;
    if (oom && oom_c == ~0ull) return h->fail(LTL_ERR_CUDA, "internal: overflow rank missing");
    if (count > 0 && materialize && !h->store_results && h->unstored_from == ~0ull) h->unstored_from = h->n_entries;
    // Matrices are written lazily: the winners' records exist now, their matrices are only needed when they
    // first serve as operands (next cost level) or are read back -- a search that ends at this level (solved,
    // ceiling) never pays for them.
    if (count > 0 && materialize && h->store_results) {
        PendingMat pm;
        pm.n_base = h->n_entries;
        pm.count = count;
        // per-record gathers waste most of each sector once matrices are long and buckets small; with short
        // matrices and dense winners the record form reads less (losers are never evaluated) -- measured both ways
        // (also for a few hundred winners: per-record phase B of BASELINE config 3's cost levels 2-4 measured slower)
        pm.tiled = h->tiled_materialize == 1 || (h->tiled_materialize < 0 && h->n >= 4096);
        if (small_screen && h->W > 1 && h->tiled_materialize < 0) {  // (a few hundred winners: neither tiles nor warps per 32 entries)
            pm.tiled = false;
            pm.small_rows = true;
        }
        if (pm.tiled) {
            pm.pieces = pieces;
            pm.total = total;
            pm.tiles = tiles;
        } else if (!small) {
            if ((rc = plan_materialize(h, pieces, total, pm.n_base, pm.count, &pm.n_seg))) return rc;
        }
        h->pending_mat.push_back(std::move(pm));
    }
    // ---- counters (reference _speedups.pyx:347-354, 372-379)
    u64 offered_c;
    if (oom) {
        out->status = LTL_S_OOM;
        out->cut_c = oom_c;
        offered_c = oom_c + 1;
        h->duplicates += oom_c - count;
    } else if (solver_c != ~0ull) {
        out->status = LTL_S_SOLVED;
        out->cut_c = solver_c;
        offered_c = solver_c + 1;
        h->duplicates += solver_c - count;
    } else {
        offered_c = (u64)total;
        h->duplicates += (u64)total - count;
    }
    if (out->status != LTL_S_DONE) {
        // statistics: tiles above the cut returned at once (or were never launched), so phase A is booked with the
        // candidates up to the cut only -- the algorithmic bytes of the roofline count work that was done
        double done_bytes = 0;
        const double B = 8.0 * (double)h->n;
        for (auto& pc : pieces) {
            if (pc.ext) continue;
            const i64 upto = std::min<i64>(pc.count, std::max<i64>(0, (i64)offered_c - pc.cbase));
            done_bytes += (double)upto * ((pc.kind == PIECE_UNARY ? 1.0 : 2.0) * B + 16.0);
        }
        h->stats[LTL_K_SCREEN].bytes += done_bytes - issued_bytes;
        h->stats[LTL_K_SCREEN].units = h->stats[LTL_K_SCREEN].units - issued_units + std::min<u64>(issued_units, offered_c);
    }
    out->admitted = count;
    const u64 gbase = h->offered;
    h->offered += offered_c;
    h->admitted += count;
    h->n_entries += count;
    if (out->status != LTL_S_DONE) {
        // keys filed at or above the cut are not members.  A search normally ends here, so the sweep over the table
        // is left to the next call that uses the table (apply_purge), if there is one.
        h->pending_purge = gbase + out->cut_c;
        h->keys_upper += (u64)total;
    } else {
        h->keys_upper += count;
    }
    return LTL_OK;
}

// LTLLEARN_DEBUG_MASKS / option "debug_masks": the reference's debug invariant (bitsem.py:46-61) on stored entries
static int check_masks(ltl_core* h, u64 first, u64 count) {
    if (!count) return LTL_OK;
    if (!h->d_dbg) CK(cudaMalloc(&h->d_dbg, 8));
    CK(cudaMemsetAsync(h->d_dbg, 0, 8, h->stream));
    const u64 groups = (first + count + 31) / 32 - first / 32;
    const u64 threads = groups * (u64)h->n * 32;
    k_check_masks<<<(unsigned)((threads + 255) / 256), 256, 0, h->stream>>>((const u64*)h->cms.base, h->d_masks, (i64)first, (i64)count,
                                                                               h->n, h->d_dbg);
    CK(cudaGetLastError());
    u64 bad = 0;
    CK(cudaMemcpyAsync(&bad, h->d_dbg, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (bad) return h->fail(LTL_ERR_INVARIANT, "characteristic bits escaped the validity mask (" + std::to_string(bad) + " words, entries " +
                                                   std::to_string(first) + ".." + std::to_string(first + count - 1) + ")");
    return LTL_OK;
}

// Phase B for every admitted-but-unwritten range.  With `sp` (the admission pass being issued) and fuse_kind != 0 it
// also screens NOT(entry) for every entry it writes: candidate not_cbase + (entry - not_i0) of that pass.
// With `store_gate` (fused launches only) the store is conditional (MaterializeParams::store_gate) and the ranges stay
// pending: the caller drops them once it knows the gate was open.
static int flush_materialize(ltl_core* h, const ScreenParams* sp, int fuse_kind, i64 not_cbase, i64 not_i0, const u64* store_gate) {
    int rc;
    for (auto& pm : h->pending_mat) {
        const u64 n_base = pm.n_base, count = pm.count;
        if ((rc = ensure_entries(h, n_base + count))) return rc;
        const double bytes = (double)count * (8.0 * (double)h->n + 16.0 + 9.0);
        if (pm.tiled) {
            // tile-shaped: the same pieces / tiles as phase A; every lane looks up its candidates' verdicts
            // (d_dest) and stores the winners, so each operand line is read once per tile
            if ((rc = ensure_pieces(h, (int)pm.pieces.size()))) return rc;
            CK(cudaStreamSynchronize(h->stream));
            memcpy(h->h_pieces, pm.pieces.data(), sizeof(Piece) * pm.pieces.size());
            CK(cudaMemcpyAsync(h->d_pieces, h->h_pieces, sizeof(Piece) * pm.pieces.size(), cudaMemcpyHostToDevice, h->stream));
            h->h2d_bytes += sizeof(Piece) * pm.pieces.size();
            ScreenParams p;
            memset(&p, 0, sizeof(p));
            p.cms = (const u64*)h->cms.base;
            p.cms_out = (u64*)h->cms.base;
            p.masks = h->d_masks;
            p.pieces = h->d_pieces;
            p.n_pieces = (int)pm.pieces.size();
            p.R = h->R;
            p.W = h->W;
            p.n_pos = h->n_pos;
            p.n_pos_lo = h->n_pos_lo;
            p.pair = h->pair ? 1 : 0;
            p.n = h->n;
            p.total_tiles = pm.tiles;
            choose_split(h, pm.tiles, &p.nsplit, &p.rows_per_split);
            p.mode = MODE_REWRITE;
            p.dest = h->d_dest;
            p.n_base = (i64)n_base;
            p.ctl = h->d_ctl;
            ScopedTimer t(h, LTL_K_MATERIALIZE, count, bytes);
            dim3 grid((unsigned)((pm.tiles * p.nsplit + LTL_WARPS_PER_CTA - 1) / LTL_WARPS_PER_CTA), 1);
            (h->pair ? ltl_launch_screen_w1p : SCREEN_FN[h->W])(p, KIND_REWRITE, grid, h->stream);
            CK(cudaGetLastError());
            continue;
        }
        MaterializeParams m;
        memset(&m, 0, sizeof(m));
        m.cms = (u64*)h->cms.base;
        m.masks = h->d_masks;
        m.R = h->R;
        m.W = h->W;
        m.n = h->n;
        m.n_base = (i64)n_base;
        m.count = (i64)count;
        m.rec_op = (const unsigned char*)h->rec_op.base;
        m.rec_lhs = (const int*)h->rec_lhs.base;
        m.rec_rhs = (const int*)h->rec_rhs.base;
        m.blk_base = h->blk_base;
        if (pm.n_seg > 0) {
            m.n_seg = pm.n_seg;
            m.seg_g0 = h->d_plan_g0;
            m.seg_goff = h->d_plan_off;
            h->plan_in_use = false;  // (the launch below is the last reader; later plans are written behind it in stream order)
        }
        if (pm.small_rows) {
            ScopedTimer t(h, LTL_K_MATERIALIZE, count, bytes);
            const dim3 grid((unsigned)((count + 3) / 4), (unsigned)((h->R + LTL_SPLIT_ROWS - 1) / LTL_SPLIT_ROWS));
            if (h->W == 2) k_materialize_small_rows<2><<<grid, 256, 0, h->stream>>>(m);
            else if (h->W == 4) k_materialize_small_rows<4><<<grid, 256, 0, h->stream>>>(m);
            else if (h->W == 8) k_materialize_small_rows<8><<<grid, 256, 0, h->stream>>>(m);
            else k_materialize_small_rows<16><<<grid, 256, 0, h->stream>>>(m);
            CK(cudaGetLastError());
            continue;
        }
        const i64 groups = (i64)((n_base + count + 31) / 32 - n_base / 32);
        choose_split(h, groups, &m.nsplit, &m.rows_per_split);
        ScreenParams none;
        memset(&none, 0, sizeof(none));
        int fk = 0;
        if (sp && fuse_kind) {  // every lane folds all rows of its entry: no row split
            m.nsplit = 1;
            m.rows_per_split = h->R;
            m.n_pos = h->n_pos;
            m.n_pos_lo = h->n_pos_lo;
            m.not_cbase = not_cbase;
            m.not_i0 = not_i0;
            m.store_gate = store_gate;
            fk = fuse_kind;
        }
        ScopedTimer t(h, LTL_K_MATERIALIZE, count, bytes + (fk ? (double)count * 16.0 : 0.0));
        dim3 grid((unsigned)((groups + LTL_WARPS_PER_CTA - 1) / LTL_WARPS_PER_CTA), (unsigned)m.nsplit);
        (h->pair ? ltl_launch_materialize_w1p : MATERIALIZE_FN[h->W])(m, fk ? *sp : none, fk, grid, h->stream);
        CK(cudaGetLastError());
        if (fk && store_gate) h->stats[LTL_K_MATERIALIZE].launches += 1;  // (the storing kernel and its evaluate-only twin)
    }
    if (store_gate) return LTL_OK;
    if (h->debug_masks)
        for (auto& pm : h->pending_mat)
            if ((rc = check_masks(h, pm.n_base, pm.count))) {
                h->pending_mat.clear();
                return rc;
            }
    h->pending_mat.clear();
    return LTL_OK;
}

// ------------------------------------------------------------------------------------------------
// level driver: units -> chunks of <= chunk_cap candidates, consecutive in enumeration order

static double steady_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int run_units(ltl_core* h, const std::vector<Unit>& units, bool check_solve, int* status, int* seg_index,
                     int64_t* li, int64_t* ri) {
    *status = LTL_S_DONE;
    *seg_index = -1;
    *li = *ri = -1;
    // Phase B of the newest cost level is due now (its matrices are first needed by this level).  When this level
    // starts with NOT over exactly those entries (it does unless negation is disabled), phase B screens NOT(entry)
    // itself while the entry's rows are in registers, and that unit gets ranks but no tiles of its own.
    i64 fuse_from = -1;
    // Candidates per pass.  When the budget has room for far fewer entries than the level has candidates, the pass that
    // exhausts it is found sooner with smaller passes (everything after the first over-budget candidate is wasted work:
    // a 150 M candidate level evaluated to admit the last 3 M entries cost 120 ms of a 215 ms search).
    i64 level_cap = h->chunk_cap;
    // A deadline is looked at between passes, like the reference's check between its 2^22-candidate chunks of 64-word
    // matrices (enumerator.py:278, 290): passes are bounded by about 2^31 matrix words so that the check comes round
    // every ~0.1 s whatever the number of rows.
    if (h->deadline_at > 0) level_cap = std::min<i64>(level_cap, std::max<i64>((i64)1 << 15, ((i64)1 << 31) / std::max<i64>(h->n, 1)));
    if (check_solve) {
        const u64 room = h->cap_entries > h->n_entries ? h->cap_entries - h->n_entries : 0;
        if (room < (u64)level_cap / 2) level_cap = std::min<i64>(level_cap, std::max<i64>((i64)room * 2, (i64)1 << 21));
    }
    if (!units.empty()) {
        if (h->fuse_not && h->W == 1 && check_solve && (h->variant == VAR_MUELLER || h->variant == VAR_NH) && !h->pending_mat.empty()) {
            const u64 pend0 = h->pending_mat.front().n_base;
            const u64 pend1 = h->pending_mat.back().n_base + h->pending_mat.back().count;
            const Unit& u0 = units[0];
            bool ok = u0.kind == PIECE_UNARY && u0.op == OP_NOT && (u64)u0.i1 == pend1 && (u64)u0.i0 <= pend0 &&
                      pend1 == h->n_entries && u0.i1 - u0.i0 <= level_cap && (i64)(pend1 - pend0) >= h->fuse_not_min;
            for (auto& pm : h->pending_mat) ok = ok && !pm.tiled;
            if (ok) fuse_from = (i64)pend0;
        }
        if (fuse_from < 0) {
            int rcf = flush_materialize(h);
            if (rcf == LTL_ERR_DEVICE_OOM) {  // the operands of this level do not fit the device: out of memory
                h->device_oom = true;
                *status = LTL_S_OOM;
                return LTL_OK;
            }
            if (rcf) return rcf;
        }
    }
    std::vector<Piece> pieces;
    size_t ui = 0;
    i64 row = units.empty() ? 0 : units[0].i0;  // next row (left index) of the current unit
    i64 col = -1;                               // >= 0: next column inside a partially emitted row
    while (ui < units.size()) {
        if (h->deadline_at > 0 && steady_seconds() > h->deadline_at) {
            *status = LTL_S_TIMEOUT;
            return LTL_OK;
        }
        pieces.clear();
        i64 total = 0, tiles = 0;
        int fused_piece = -1;
        const i64 cap = level_cap;
        while (ui < units.size() && total < cap) {
            const Unit& u = units[ui];
            const i64 room = cap - total;
            bool unit_done = false;
            if (u.kind == PIECE_UNARY) {
                i64 take = std::min(room, u.i1 - row);
                const bool fused_part = fuse_from >= 0 && ui == 0 && row >= fuse_from;
                if (fuse_from >= 0 && ui == 0 && row < fuse_from) take = std::min(take, fuse_from - row);  // written part first
                push_piece(h, pieces, total, tiles, u, row, row + take, -1, -1, PIECE_UNARY, fused_part);
                if (fused_part) fused_piece = (int)pieces.size() - 1;
                row += take;
                unit_done = row == u.i1;
            } else {
                // columns of row `row`: [cstart, u.j1)
                const i64 c0 = u.kind == PIECE_RECT ? u.j0 : row + 1;
                if (col >= 0) {  // finish a partially emitted row
                    const i64 take = std::min(room, u.j1 - col);
                    push_piece(h, pieces, total, tiles, u, row, row + 1, col, col + take, PIECE_RECT);
                    col += take;
                    if (col == u.j1) {
                        col = -1;
                        row++;
                    }
                    unit_done = row == u.i1;
                } else {
                    i64 rows_fit;
                    if (u.kind == PIECE_RECT) {
                        rows_fit = std::min(u.i1 - row, room / (u.j1 - u.j0));
                    } else {
                        const u64 m = (u64)(u.j1 - 1 - row);
                        i64 lo = 0, hi = u.i1 - row;
                        while (lo < hi) {
                            i64 mid = (lo + hi + 1) >> 1;
                            if (tri_before((u64)mid, m) <= (u64)room) lo = mid;
                            else hi = mid - 1;
                        }
                        rows_fit = lo;
                    }
                    if (rows_fit > 0) {
                        if (u.kind == PIECE_RECT) push_piece(h, pieces, total, tiles, u, row, row + rows_fit, u.j0, u.j1, PIECE_RECT);
                        else push_piece(h, pieces, total, tiles, u, row, row + rows_fit, -1, u.j1, PIECE_TRI);
                        row += rows_fit;
                        unit_done = row == u.i1;
                    } else if (total == 0) {  // a single row exceeds the chunk: emit it in column runs
                        col = c0;
                        continue;
                    } else {
                        break;  // close the chunk, the row starts the next one
                    }
                }
            }
            if (unit_done) {
                ui++;
                if (ui < units.size()) row = units[ui].i0;
                col = -1;
            }
        }
        ChunkOut co;
        int rc = run_chunk(h, pieces, total, tiles, MODE_INSERT, check_solve, true, &co, fused_piece);
        if (rc == LTL_ERR_DEVICE_OOM && fused_piece >= 0) {  // phase B of the operands did not fit the device
            h->device_oom = true;
            *status = LTL_S_OOM;
            return LTL_OK;
        }
        if (rc) return rc;
        if (co.status != LTL_S_DONE) {
            *status = co.status;
            if (co.status == LTL_S_SOLVED) {
                size_t pi = 0;
                for (size_t k = 0; k < pieces.size(); k++)
                    if ((u64)pieces[k].cbase <= co.cut_c) pi = k;
                i64 i, j;
                piece_unrank(pieces[pi], co.cut_c, &i, &j);
                *li = i;
                *ri = j;
                *seg_index = pieces[pi].seg;
            }
            return LTL_OK;
        }
    }
    return LTL_OK;
}

static i64 unit_count(const Unit& u) {
    if (u.kind == PIECE_UNARY) return u.i1 - u.i0;
    if (u.kind == PIECE_RECT) return (u.i1 - u.i0) * (u.j1 - u.j0);
    return (i64)tri_before((u64)(u.i1 - u.i0), (u64)(u.j1 - 1 - u.i0));
}

// Pieces covering exactly the level ranks [lo, hi) of the unit list, in rank order (piece cbase = rank - lo).
static void plan_range(ltl_core* h, const std::vector<Unit>& units, i64 lo, i64 hi, std::vector<Piece>& pieces,
                       i64& total, i64& tiles) {
    i64 ustart = 0;
    for (const Unit& u : units) {
        const i64 cnt = unit_count(u);
        const i64 a = std::max(lo, ustart) - ustart, b = std::min(hi, ustart + cnt) - ustart;
        ustart += cnt;
        if (a >= b) continue;
        if (u.kind == PIECE_UNARY) {
            push_piece(h, pieces, total, tiles, u, u.i0 + a, u.i0 + b, -1, -1, PIECE_UNARY);
        } else if (u.kind == PIECE_RECT) {
            const i64 nj = u.j1 - u.j0;
            i64 ra = a / nj, ca = a % nj;
            const i64 rb = b / nj, cb = b % nj;
            if (ra == rb) {
                push_piece(h, pieces, total, tiles, u, u.i0 + ra, u.i0 + ra + 1, u.j0 + ca, u.j0 + cb, PIECE_RECT);
                continue;
            }
            if (ca > 0) {
                push_piece(h, pieces, total, tiles, u, u.i0 + ra, u.i0 + ra + 1, u.j0 + ca, u.j1, PIECE_RECT);
                ra++;
            }
            if (rb > ra) push_piece(h, pieces, total, tiles, u, u.i0 + ra, u.i0 + rb, u.j0, u.j1, PIECE_RECT);
            if (cb > 0) push_piece(h, pieces, total, tiles, u, u.i0 + rb, u.i0 + rb + 1, u.j0, u.j0 + cb, PIECE_RECT);
        } else {
            Piece t;
            memset(&t, 0, sizeof(t));
            t.kind = PIECE_TRI;
            t.i0 = u.i0;
            t.i1 = u.i1;
            t.j1 = u.j1;
            i64 ia, ja, ib, jb;
            piece_unrank(t, (u64)a, &ia, &ja);
            if (b < cnt) piece_unrank(t, (u64)b, &ib, &jb);
            else {
                ib = u.i1;
                jb = u.i1 + 1;
            }
            // [ (ia, ja), (ib, jb) ) in row-major order; row i holds columns (i, j1)
            if (ia == ib) {
                push_piece(h, pieces, total, tiles, u, ia, ia + 1, ja, jb, PIECE_RECT);
                continue;
            }
            if (ja > ia + 1) {
                push_piece(h, pieces, total, tiles, u, ia, ia + 1, ja, u.j1, PIECE_RECT);
                ia++;
            }
            if (ib > ia) push_piece(h, pieces, total, tiles, u, ia, ib, -1, u.j1, PIECE_TRI);
            if (ib < u.i1 && jb > ib + 1) push_piece(h, pieces, total, tiles, u, ib, ib + 1, ib + 1, jb, PIECE_RECT);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// single-matrix paths (add_entry / contains / fingerprint_of)

// half-width store: uint64[R] rows (positions in the high half) <-> ceil(R / 2) words holding rows 2v | 2v + 1
static void pack_pairs(const uint64_t* rows, int R, u64* out) {
    for (int v = 0; 2 * v < R; v++)
        out[v] = (rows[2 * v] & 0xFFFFFFFF00000000ull) | (2 * v + 1 < R ? rows[2 * v + 1] >> 32 : 0ull);
}
static void unpack_pairs(const u64* words, int R, uint64_t* out) {
    for (int v = 0; 2 * v < R; v++) {
        out[2 * v] = words[v] & 0xFFFFFFFF00000000ull;
        if (2 * v + 1 < R) out[2 * v + 1] = words[v] << 32;
    }
}

static int stage_matrix(ltl_core* h, const uint64_t* cm, i64 e) {
    int rc;
    if ((rc = ensure_entries(h, (u64)e + 1))) return rc;
    CK(cudaStreamSynchronize(h->stream));  // h_stage may still be in flight
    if (h->pair) pack_pairs(cm, h->R_api, h->h_stage);
    else memcpy(h->h_stage, cm, (size_t)h->n * 8);
    CK(cudaMemcpyAsync(h->d_stage, h->h_stage, (size_t)h->n * 8, cudaMemcpyHostToDevice, h->stream));
    h->h2d_bytes += (size_t)h->n * 8;
    ScopedTimer t(h, LTL_K_MISC, 1, 16.0 * (double)h->n);
    k_import<<<(unsigned)((h->n + 255) / 256), 256, 0, h->stream>>>(h->d_stage, (u64*)h->cms.base, e, h->n);
    CK(cudaGetLastError());
    return LTL_OK;
}

static int single_chunk(ltl_core* h, i64 e, int mode, ChunkOut* co) {
    std::vector<Piece> pieces;
    i64 total = 0, tiles = 0;
    Unit u{PIECE_UNARY, OP_IDENT, 0, e, e + 1, -1, -1};
    push_piece(h, pieces, total, tiles, u, e, e + 1, -1, -1, PIECE_UNARY);
    return run_chunk(h, pieces, total, tiles, mode, false, false, co);
}

// ------------------------------------------------------------------------------------------------
// fingerprint deposits for the bit-gathering variants

static int build_deposits(ltl_core* h, const int32_t* proj_rows, const int32_t* proj_offs, int n_proj, std::vector<Deposit>& deps) {
    if (h->variant == VAR_GATHER) {  // reference _speedups.pyx:188-195: bit b of the projection -> bit 125 - b
        for (int b = 0; b < n_proj; b++) {
            const int r = proj_rows[b], off = proj_offs[b];
            if (r < 0 || r >= h->R || off < 0 || off >= 64 * h->W) return h->fail(LTL_ERR_ARG, "projection outside the matrix");
            Deposit d;
            d.k = (u32)(r * h->W + (off >> 6));
            d.rsh = (u32)(63 - (off & 63));
            d.mask = 1;
            d.pos = (u32)(125 - b);
            d.pad = 0;
            deps.push_back(d);
        }
    } else if (h->variant == VAR_FKP) {  // reference _speedups.pyx:205-222: first fkp_bits positions of every row
        if (h->fkp_bits < 1 || h->fkp_bits > 64) return h->fail(LTL_ERR_ARG, "fkp_bits must lie in [1, 64]");
        int used = 0;
        for (int r = 0; r < h->R; r++) {
            int nb = std::min(126 - used, h->fkp_bits);
            if (nb <= 0) break;
            Deposit d;
            d.k = (u32)(r * h->W);
            d.rsh = (u32)(64 - nb);
            d.mask = nb >= 64 ? ~0ull : ((1ull << nb) - 1ull);
            d.pos = (u32)(126 - used - nb);
            d.pad = 0;
            deps.push_back(d);
            used += nb;
        }
    }
    std::stable_sort(deps.begin(), deps.end(), [](const Deposit& a, const Deposit& b) { return a.k < b.k; });
    return LTL_OK;
}

// ------------------------------------------------------------------------------------------------
// C ABI

struct PackScratch {
    void* buf = nullptr;
    size_t cap = 0;
    cudaStream_t st = nullptr;
};

extern "C" {

int ltl_pack_traces(const uint16_t* chars, const int64_t* lengths, int64_t R, int L, int n_props, int W, int device,
                    uint64_t* masks_out, uint64_t* atoms_out) {
    g_create_error.clear();
    auto bad = [&](const char* m) {
        g_create_error = m;
        return LTL_ERR_ARG;
    };
    if (R < 0 || L < 0 || W < 1 || W > LTL_MAX_W || n_props < 1 || n_props > 16) return bad("pack: bad shape");
    if (L > 64 * W) return bad("pack: traces do not fit W words");
    if (R == 0) return LTL_OK;
    if (!chars || !lengths || !masks_out || !atoms_out) return bad("pack: null buffer");
    auto cuda_fail = [&](cudaError_t e) {
        g_create_error = std::string("pack: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return LTL_ERR_CUDA;
    };
    cudaError_t e;
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e);
    const int Lpad = 64 * W;  // device rows are padded to whole words so that the 16-byte loads stay in bounds
    const size_t words = (size_t)R * W;
    // one grow-only device scratch and one stream per device, kept for the life of the process: a learn() call makes
    // no memory-management call for packing (cudaMalloc / cudaFree synchronise the whole device)
    static std::mutex mu;
    static PackScratch scratch[LTL_MAX_DEVICES];
    if (device < 0 || device >= LTL_MAX_DEVICES) return bad("pack: bad device");
    std::lock_guard<std::mutex> lock(mu);
    PackScratch& ps = scratch[device];
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t b_chars = up((size_t)R * Lpad * 2), b_len = up((size_t)R * 8), b_out = up(words * 8 * (size_t)(n_props + 1));
    if (!ps.st && (e = cudaStreamCreateWithFlags(&ps.st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e);
    if (ps.cap < b_chars + b_len + b_out) {
        if (ps.buf) cudaFree(ps.buf);
        ps.buf = nullptr;
        ps.cap = 0;
        if ((e = cudaMalloc(&ps.buf, b_chars + b_len + b_out)) != cudaSuccess) return cuda_fail(e);
        ps.cap = b_chars + b_len + b_out;
    }
    cudaStream_t st = ps.st;
    uint16_t* d_chars = (uint16_t*)ps.buf;
    i64* d_len = (i64*)((char*)ps.buf + b_chars);
    u64* d_out = (u64*)((char*)ps.buf + b_chars + b_len);
    if (L == Lpad) {
        e = cudaMemcpyAsync(d_chars, chars, (size_t)R * L * 2, cudaMemcpyHostToDevice, st);
    } else {
        if ((e = cudaMemsetAsync(d_chars, 0, (size_t)R * Lpad * 2, st)) != cudaSuccess) return cuda_fail(e);
        e = L ? cudaMemcpy2DAsync(d_chars, (size_t)Lpad * 2, chars, (size_t)L * 2, (size_t)L * 2, (size_t)R, cudaMemcpyHostToDevice, st)
              : cudaSuccess;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemcpyAsync(d_len, lengths, (size_t)R * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e);
    const unsigned nb = (unsigned)((words + 255) / 256);
    if (n_props <= 4) k_pack<4><<<nb, 256, 0, st>>>(d_chars, d_len, R, L, Lpad, W, n_props, d_out, d_out + words);
    else if (n_props <= 8) k_pack<8><<<nb, 256, 0, st>>>(d_chars, d_len, R, L, Lpad, W, n_props, d_out, d_out + words);
    else k_pack<16><<<nb, 256, 0, st>>>(d_chars, d_len, R, L, Lpad, W, n_props, d_out, d_out + words);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemcpyAsync(masks_out, d_out, words * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemcpyAsync(atoms_out, d_out + words, words * 8 * (size_t)n_props, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
    return LTL_OK;
}

int ltl_abi_version(void) { return LTL_ABI_VERSION; }

int ltl_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return LTL_ERR_CUDA;
    }
    return n;
}

const char* ltl_core_last_error(const ltl_core* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void ltl_core_destroy(ltl_core* h) {
    if (!h) return;
    if (h->device >= 0) {
        cudaSetDevice(h->device);
        if (h->stream) cudaStreamSynchronize(h->stream);
        drain_events(h);
        if (h->d_dbg) cudaFree(h->d_dbg);
        cudaFree(h->d_subtree);
        cudaFree(h->d_route_hist);
        cudaFree(h->d_route_off);
        for (auto& ev : h->part_ev)
            if (ev) cudaEventDestroy(ev);
        cudaFree(h->d_plan_g0);
        cudaFree(h->d_plan_cnt);
        cudaFree(h->d_plan_off);
        cudaFree(h->d_plan_fams);
        cudaGetLastError();
        pool_give(*static_cast<Arena*>(h));
    }
    delete h;
}

}  // extern "C"

// masks: host length masks, or null with `tr`: the masks packed on the device by ltl_traces_pack
static int core_create_impl(const uint64_t* masks, const ltl_traces* tr, int R, int W, int n_pos, int err_max, int variant,
                            const int32_t* proj_rows, const int32_t* proj_offs, int n_proj, int fkp_bits, int mask_k,
                            uint64_t budget_bytes, int device, ltl_core** out) {
    if (!out) return LTL_ERR_ARG;
    *out = nullptr;
    auto bad = [&](const char* m) {
        g_create_error = m;
        return LTL_ERR_ARG;
    };
    if ((!masks && !tr) || R < 1) return bad("need at least one row");
    if (W < 1 || W > LTL_MAX_W) return bad("words per row must lie in [1, 16]");
    if (n_pos < 0 || n_pos > R) return bad("n_pos outside [0, R]");
    if (variant < 0 || variant > VAR_NH32) return bad("unknown fingerprint variant");
    if (variant == VAR_NH32 && W != 1) return bad("the half-width variant (NH32) needs one word per row");
    if (n_proj < 0 || n_proj > 126) return bad("projection wider than the fingerprint");  // reference _speedups.pyx:92-93
    if (mask_k < 0 || mask_k > 126) return bad("mask_k outside [0, 126]");
    if ((int64_t)R * W > (int64_t)1 << 31) return bad("matrix too large");
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev < 1) {
        g_create_error = std::string("no usable CUDA device: ") + cudaGetErrorString(ce);
        cudaGetLastError();
        return LTL_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) return bad("device index out of range");
    ltl_core* h = new ltl_core();
    h->device = device;
    h->R_api = R;
    h->n_api = (i64)R * W;
    h->pair = variant == VAR_NH32;
    h->R = h->pair ? (R + 1) / 2 : R;
    h->W = W;
    h->n = (i64)h->R * W;
    h->n_pos = h->pair ? (n_pos + 1) / 2 : n_pos;
    h->n_pos_lo = h->pair ? n_pos / 2 : n_pos;
    h->err_max = err_max;
    h->variant = h->pair ? VAR_NH : variant;
    h->fkp_bits = fkp_bits;
    h->mask_k = mask_k;
    h->budget = budget_bytes;
    h->entry_bytes = (u64)h->n_api * 8 + 16;  // reference _speedups.pyx:100 (logical: one 64-bit word per row)
    int rc = LTL_OK;
    auto boot = [&]() -> int {
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device));
        Arena pooled;
        const bool reused = pool_enabled() && pool_take(device, pooled);
        if (reused) static_cast<Arena&>(*h) = pooled;
        h->device = device;
        if (!h->stream) CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        // cudaMemGetInfo stalls for milliseconds now and then (measured: up to 80 ms with tens of GB mapped), so a core
        // that starts from a pooled arena sizes its (virtual) reservations from the device's total memory instead;
        // physical exhaustion is detected where pages are mapped, not here
        static size_t total_mem[LTL_MAX_DEVICES];
        size_t free_b = 0, total_b = 0;
        if (reused && device < LTL_MAX_DEVICES && total_mem[device]) {
            free_b = total_b = total_mem[device];
        } else {
            CK(cudaMemGetInfo(&free_b, &total_b));
            if (device < LTL_MAX_DEVICES) total_mem[device] = total_b;
            free_b += h->cms.mapped;  // a pooled arena's pages are ours to reuse
        }
        // admissions allowed by the logical budget: OOM when admitted*eb + eb > budget (reference _speedups.pyx:252-253)
        // The budget is LOGICAL, like the reference's: admissions are counted, and because matrices are written
        // lazily the entries of the level a search ends in never occupy memory.  Physical exhaustion is reported
        // when matrices have to be written (flush_materialize -> LTL_S_OOM from the screening call).
        u64 logical = h->budget / h->entry_bytes;
        h->cap_entries = std::min<u64>(logical, (1ull << 31) - 64);
        const double per_entry = 8.0 * (double)h->n + 9.0;
        const u64 physical = (u64)((double)(free_b > (1ull << 30) ? free_b - (1ull << 30) : 0) / per_entry);
        const u64 cap_groups = (std::min<u64>(h->cap_entries, physical + 64) + 63) / 32;
        // virtual reservations are generous and uniform so that pooled arenas fit the next core
        auto reserve = [&](GrowBuf& g, size_t need, size_t floor_bytes) {
            need = std::max(need, floor_bytes);
            if (g.base && g.reserved >= need) return;
            g.release();
            g.init(device, need);
        };
        reserve(h->cms, (size_t)cap_groups * 32 * (size_t)h->n * 8, (size_t)256 << 30);
        reserve(h->rec_op, (size_t)cap_groups * 32, (size_t)2 << 30);
        reserve(h->rec_lhs, (size_t)cap_groups * 32 * 4, (size_t)8 << 30);
        reserve(h->rec_rhs, (size_t)cap_groups * 32 * 4, (size_t)8 << 30);
        if (h->masks_cap < h->n) {
            cudaFree(h->d_masks);
            h->d_masks = nullptr;
            h->masks_cap = 0;
            CK(cudaMalloc(&h->d_masks, (size_t)h->n * 8));
            h->masks_cap = h->n;
        }
        if (h->stage_cap < h->n) {
            cudaFree(h->d_stage);
            cudaFreeHost(h->h_stage);
            h->d_stage = h->h_stage = nullptr;
            h->stage_cap = 0;
            CK(cudaMalloc(&h->d_stage, (size_t)h->n * 8));
            CK(cudaMallocHost(&h->h_stage, (size_t)h->n * 8));
            h->stage_cap = h->n;
        }
        if (tr) {  // the masks are in HBM already (the traces' stream is idle: ltl_traces_pack waits for its kernel)
            if (h->pair) k_pack_pairs<<<(unsigned)((h->n + 255) / 256), 256, 0, h->stream>>>(tr->d_masks, h->R_api, h->d_masks, h->n);
            else CK(cudaMemcpyAsync(h->d_masks, tr->d_masks, (size_t)h->n * 8, cudaMemcpyDeviceToDevice, h->stream));
            CK(cudaGetLastError());
        } else {
            if (h->pair) pack_pairs(masks, h->R_api, h->h_stage);
            else memcpy(h->h_stage, masks, (size_t)h->n * 8);  // pinned staging: the copy below is truly asynchronous
            CK(cudaMemcpyAsync(h->d_masks, h->h_stage, (size_t)h->n * 8, cudaMemcpyHostToDevice, h->stream));
            h->h2d_bytes += (size_t)h->n * 8;
        }
        std::vector<Deposit> deps;
        int r2 = build_deposits(h, proj_rows, proj_offs, n_proj, deps);
        if (r2) return r2;
        h->n_dep = (int)deps.size();
        if (h->deps_cap < std::max(1, h->n_dep)) {
            cudaFree(h->d_deps);
            h->d_deps = nullptr;
            h->deps_cap = 0;
            CK(cudaMalloc(&h->d_deps, sizeof(Deposit) * std::max<size_t>(1, deps.size())));
            h->deps_cap = std::max(1, h->n_dep);
        }
        if (!deps.empty()) {
            CK(cudaMemcpyAsync(h->d_deps, deps.data(), sizeof(Deposit) * deps.size(), cudaMemcpyHostToDevice, h->stream));
            CK(cudaStreamSynchronize(h->stream));
        }
        if (!h->sub_ev[0]) {
            CK(cudaEventCreateWithFlags(&h->sub_ev[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->sub_ev[1], cudaEventDisableTiming));
            CK(cudaMallocHost(&h->h_solver, 2 * sizeof(u64)));
        }
        if (!h->d_ctl) CK(cudaMalloc(&h->d_ctl, sizeof(Ctl)));
        if (!h->h_ctl) CK(cudaMallocHost(&h->h_ctl, sizeof(Ctl)));
        if (h->table) {  // pooled table: keep its size (no rehash in steady state), forget its keys
            CK(cudaMemsetAsync(h->table, 0xFF, h->table_cap * sizeof(Slot), h->stream));
            return LTL_OK;
        }
        return ensure_table(h, 1);
    };
    rc = boot();
    if (rc) {
        g_create_error = h->err;
        ltl_core_destroy(h);
        return rc;
    }
    if (getenv("LTLLEARN_DEBUG_MASKS")) h->debug_masks = true;  // the reference's switch (bitsem.py:48)
    *out = h;
    return LTL_OK;
}

extern "C" {

int ltl_core_create(const uint64_t* masks, int R, int W, int n_pos, int err_max, int variant, const int32_t* proj_rows,
                    const int32_t* proj_offs, int n_proj, int fkp_bits, int mask_k, uint64_t budget_bytes, int device,
                    ltl_core** out) {
    if (!masks) {
        g_create_error = "need at least one row";
        return LTL_ERR_ARG;
    }
    return core_create_impl(masks, nullptr, R, W, n_pos, err_max, variant, proj_rows, proj_offs, n_proj, fkp_bits, mask_k,
                            budget_bytes, device, out);
}

int ltl_core_create_on_traces(ltl_traces* t, int err_max, int variant, const int32_t* proj_rows, const int32_t* proj_offs,
                              int n_proj, int fkp_bits, int mask_k, uint64_t budget_bytes, ltl_core** out) {
    if (!t || !t->n_props) {
        g_create_error = "create_on_traces: the traces are not packed (ltl_traces_pack)";
        return LTL_ERR_ARG;
    }
    if (t->R > 0x7FFFFFFF) {
        g_create_error = "create_on_traces: too many rows";
        return LTL_ERR_ARG;
    }
    int rc = core_create_impl(nullptr, t, (int)t->R, t->W, (int)t->n_pos, err_max, variant, proj_rows, proj_offs, n_proj, fkp_bits,
                              mask_k, budget_bytes, t->device, out);
    return rc;
}

#define ENTER(h)                              \
    if (!(h)) return LTL_ERR_ARG;             \
    {                                         \
        cudaError_t e0_ = cudaSetDevice((h)->device); \
        if (e0_ != cudaSuccess) return (h)->cuda_fail(e0_, "cudaSetDevice"); \
    }

int ltl_core_add_entry(ltl_core* h, const uint64_t* cm, int op, int lhs, int rhs, int64_t* index_out) {
    ENTER(h);
    if (!cm || !index_out) return h->fail(LTL_ERR_ARG, "null argument");
    *index_out = -1;
    const i64 e = (i64)h->n_entries;
    int rc;
    if ((rc = stage_matrix(h, cm, e))) return rc;
    if (h->debug_masks && (rc = check_masks(h, (u64)e, 1))) return rc;
    ChunkOut co;
    if ((rc = single_chunk(h, e, MODE_INSERT, &co))) return rc;
    if (co.status == LTL_S_OOM) return h->fail(LTL_ERR_BUDGET, "memory budget exhausted");
    if (co.admitted == 1) {
        ScopedTimer t(h, LTL_K_MISC, 1, 9.0);
        k_set_record<<<1, 1, 0, h->stream>>>((unsigned char*)h->rec_op.base, (int*)h->rec_lhs.base, (int*)h->rec_rhs.base, e, op,
                                             lhs, rhs);
        CK(cudaGetLastError());
        *index_out = e;
    }
    return LTL_OK;
}

int ltl_core_add_atom(ltl_core* h, ltl_traces* t, int prop, int negated, int op, int lhs, int rhs, int64_t* index_out) {
    ENTER(h);
    if (!t || !index_out) return h->fail(LTL_ERR_ARG, "null argument");
    *index_out = -1;
    if (t->device != h->device || t->R * t->W != h->n_api || prop < 0 || prop >= t->n_props)
        return h->fail(LTL_ERR_ARG, "add_atom: the traces do not belong to this core (device, shape or proposition)");
    const i64 e = (i64)h->n_entries;
    int rc;
    if ((rc = ensure_entries(h, (u64)e + 1))) return rc;
    {
        ScopedTimer tm(h, LTL_K_MISC, 1, 16.0 * (double)h->n);
        k_import_dev<<<(unsigned)((h->n + 255) / 256), 256, 0, h->stream>>>(t->d_atoms + (size_t)prop * (size_t)h->n_api, t->d_masks,
                                                                              negated ? 1 : 0, h->pair ? 1 : 0, h->R_api,
                                                                              (u64*)h->cms.base, e, h->n);
    }
    CK(cudaGetLastError());
    ChunkOut co;
    if ((rc = single_chunk(h, e, MODE_INSERT, &co))) return rc;
    if (co.status == LTL_S_OOM) return h->fail(LTL_ERR_BUDGET, "memory budget exhausted");
    if (co.admitted == 1) {
        ScopedTimer tm(h, LTL_K_MISC, 1, 9.0);
        k_set_record<<<1, 1, 0, h->stream>>>((unsigned char*)h->rec_op.base, (int*)h->rec_lhs.base, (int*)h->rec_rhs.base, e, op,
                                             lhs, rhs);
        CK(cudaGetLastError());
        *index_out = e;
    }
    return LTL_OK;
}

int ltl_core_run_level(ltl_core* h, const ltl_segment* segs, int n_segs, int* status, int* seg_index, int64_t* li,
                       int64_t* ri) {
    ENTER(h);
    if (n_segs < 0 || (n_segs && !segs) || !status || !seg_index || !li || !ri) return h->fail(LTL_ERR_ARG, "null argument");
    std::vector<Unit> units;
    int rc = expand_segments(h, segs, n_segs, units);
    if (rc) return rc;
    return run_units(h, units, true, status, seg_index, li, ri);
}

// The first cost levels of a search in ONE launch (levels.cuh), while they are small: fills the stats rows of the levels it
// completed, moves the bucket table and the core's counters on, and returns in *next_cost the level the host-driven loop
// continues with (with *status == LTL_S_SOLVED: the level that solved).  Declines (next_cost = first_cost, nothing
// changed) whenever the core is not in the plain state the kernel assumes.
static int run_levels_device(ltl_core* h, const int32_t op_cost[8], uint32_t op_mask, std::vector<std::pair<i64, i64>>& bucket,
                             std::vector<char>& known, int first_cost, int ceiling, int store_last_level, ltl_level_stats* rows,
                             int* n_rows, int* status, int* op, int64_t* li, int64_t* ri, int* next_cost) {
    *next_cost = first_cost;
    if (!h->device_levels || !h->small_screen || !h->small_admit || h->W != 1 || h->pair || h->exchange || h->force_split ||
        h->debug_masks || !h->store_results || h->unstored_from != ~0ull || h->levels_max_work <= 0 || h->blk_base != 0 ||
        h->chunk_cap < LTL_LV_MAX_TOTAL)
        return LTL_OK;
    const int stop_cost = std::min(ceiling, LTL_LV_MAX_COST);
    if (first_cost >= stop_cost || first_cost < 1) return LTL_OK;
    int rc;
    LevelsParams P;
    memset(&P, 0, sizeof(P));
    P.sp.R = h->R;
    P.sp.n = h->n;
    P.first_cost = first_cost;
    P.stop_cost = stop_cost;
    P.nostore_cost = store_last_level ? -1 : ceiling - 1;  // the last level of a search is not stored unless asked for
    for (int k = 0; k < 8; k++) P.op_cost[k] = op_cost[k];
    P.op_mask = op_mask;
    P.max_total = LTL_LV_MAX_TOTAL;
    P.max_work = h->levels_max_work;
    const u64 room = h->cap_entries > h->n_entries ? h->cap_entries - h->n_entries : 0;
    // store mapped ahead of the launch: what the levels it may run can admit, bounded in bytes
    const u64 ahead = std::min<u64>(room, std::max<u64>(4096, std::min<u64>(4 * (u64)P.max_total, ((u64)256 << 20) / (8 * (u64)h->n))));
    P.entry_cap = h->n_entries + ahead;
    {   // is the first level one for the device at all?  (same planner, on the host)
        static thread_local std::vector<Piece> scratch(LTL_LV_MAX_PIECES);
        i64 bf[LTL_LV_MAX_COST], be[LTL_LV_MAX_COST];
        for (int k = 0; k < LTL_LV_MAX_COST; k++) {
            bf[k] = k < (int)bucket.size() ? bucket[(size_t)k].first : 0;
            be[k] = k < (int)bucket.size() ? bucket[(size_t)k].second : 0;
        }
        int np = 0;
        i64 total = 0;
        double bytes = 0;
        P.table_cap = ~0ull;
        if (!lv_plan(first_cost, P.op_cost, P.op_mask, bf, be, scratch.data(), LTL_LV_MAX_PIECES, &np, &total, &bytes, 0.0) ||
            !lv_fits(P, total, h->n_entries, h->keys_upper))
            return LTL_OK;
    }
    if (h->deadline_at > 0 && steady_seconds() > h->deadline_at) {
        *status = LTL_S_TIMEOUT;
        return LTL_OK;
    }
    if ((rc = flush_materialize(h))) return rc == LTL_ERR_DEVICE_OOM ? LTL_OK : rc;
    if ((rc = apply_purge(h))) return rc;
    if ((rc = ensure_table(h, h->keys_upper + 4 * (u64)P.max_total))) return rc == LTL_ERR_DEVICE_OOM ? LTL_OK : rc;
    if ((rc = ensure_scratch(h, P.max_total))) return rc;
    if ((rc = ensure_acc(h, P.max_total))) return rc;
    if ((rc = ensure_entries(h, P.entry_cap))) return rc == LTL_ERR_DEVICE_OOM ? LTL_OK : rc;
    if (!h->d_lv) {
        CK(cudaMalloc(&h->d_lv, sizeof(LevelsState)));
        CK(cudaMallocHost(&h->h_lv, sizeof(LevelsState)));
    }
    if (h->R > LTL_SPLIT_ROWS) {
        // rows in several hash blocks: the blocks' sums meet in the partial-sum array.  `acc_dirty == false` only promises
        // zeros in the part small host-driven passes use (LTL_SMALL_ADMIT candidates); a level here may be larger, and a
        // pooled arena remembers the sums of an earlier search beyond that part (found by scripts/levels_diff.py)
        CK(cudaMemsetAsync(h->d_acc, 0, (size_t)P.max_total * 24, h->stream));
        if (h->acc_cap <= P.max_total) h->acc_dirty = false;  // (the kernel leaves the sums it consumed zeroed, like k_admit_small)
    }
    CK(cudaMemsetAsync(h->d_ctl, 0xFF, sizeof(Ctl), h->stream));
    LevelsState& S = *h->h_lv;
    memset(&S, 0, sizeof(S));
    S.n_entries = h->n_entries;
    S.offered = h->offered;
    S.admitted = h->admitted;
    S.duplicates = h->duplicates;
    S.keys_upper = h->keys_upper;
    S.next_cost = first_cost;
    S.status = LTL_S_DONE;
    S.unstored_from = ~0ull;
    for (int k = 0; k < LTL_LV_MAX_COST && k < (int)bucket.size(); k++) {
        S.bucket_first[k] = bucket[(size_t)k].first;
        S.bucket_end[k] = bucket[(size_t)k].second;
        S.known[k] = known[(size_t)k];
    }
    CK(cudaMemcpyAsync(h->d_lv, h->h_lv, sizeof(LevelsState), cudaMemcpyHostToDevice, h->stream));
    h->h2d_bytes += sizeof(LevelsState);
    P.sp.cms = (const u64*)h->cms.base;
    P.sp.masks = h->d_masks;
    P.sp.W = 1;
    P.sp.n_pos = h->n_pos;
    P.sp.n_pos_lo = h->n_pos_lo;
    P.sp.err_max = h->err_max;
    P.sp.variant = h->variant;
    P.sp.mask_k = h->mask_k;
    P.sp.n_dep = h->n_dep;
    P.sp.deps = h->d_deps;
    P.sp.mode = MODE_INSERT;
    P.sp.check_solve = 1;
    P.sp.table = h->table;
    P.sp.table_mask = h->table_cap - 1;
    P.sp.slot = h->d_slot;
    P.sp.acc = h->d_acc;
    P.sp.ctl = h->d_ctl;
    P.sp.owner_world = 1;
    P.cms_w = (u64*)h->cms.base;
    P.rec_op = (unsigned char*)h->rec_op.base;
    P.rec_lhs = (int*)h->rec_lhs.base;
    P.rec_rhs = (int*)h->rec_rhs.base;
    P.st = h->d_lv;
    P.table_cap = h->table_cap;
    const auto t0 = std::chrono::steady_clock::now();
    {
        ScopedTimer t(h, LTL_K_LEVELS, 0, 0.0);
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3((unsigned)h->levels_ctas, 1, 1);
        cfg.blockDim = dim3(LTL_LV_CTA, 1, 1);
        cfg.stream = h->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)h->levels_ctas;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (h->variant == VAR_MUELLER) CK(cudaLaunchKernelEx(&cfg, k_levels<KIND_MUELLER>, P));
        else if (h->variant == VAR_NH) CK(cudaLaunchKernelEx(&cfg, k_levels<KIND_NH>, P));
        else CK(cudaLaunchKernelEx(&cfg, k_levels<KIND_BITS>, P));
    }
    CK(cudaMemcpyAsync(h->h_lv, h->d_lv, sizeof(LevelsState), cudaMemcpyDeviceToHost, h->stream));
    {
        HostTimer ht(&h->sync_ms);
        CK(cudaStreamSynchronize(h->stream));
    }
    h->d2h_bytes += sizeof(LevelsState);
    drain_events(h);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (getenv("LTL_LEVELS_TRACE")) {  // where the launch spent its time (device clock, ns since the level began)
        for (int k = 0; k < S.n_rows; k++) {
            const u64* t = S.t_ns[k];
            fprintf(stderr, "levels: cost %d offered %llu admitted %llu  planned %llu screened %llu admitted %llu booked %llu stored %llu ns\n",
                    S.rows[k].cost, (unsigned long long)S.rows[k].offered, (unsigned long long)S.rows[k].admitted,
                    (unsigned long long)(t[1] - t[0]), (unsigned long long)(t[2] - t[0]), (unsigned long long)(t[3] - t[0]),
                    (unsigned long long)(t[4] - t[0]), (unsigned long long)(t[5] ? t[5] - t[0] : 0));
        }
        fprintf(stderr, "levels: launch to state read back %.1f us, next cost %d (stop %d, unstored level %d)\n", 1e3 * ms, S.next_cost,
                P.stop_cost, P.nostore_cost);
        if (S.status == LTL_S_DONE && S.next_cost < P.stop_cost) {  // why the hand-over?
            static thread_local std::vector<Piece> scratch(LTL_LV_MAX_PIECES);
            int np = 0;
            i64 total = 0;
            double bytes = 0;
            const bool planned = lv_plan(S.next_cost, P.op_cost, P.op_mask, S.bucket_first, S.bucket_end, scratch.data(), LTL_LV_MAX_PIECES,
                                         &np, &total, &bytes, 0.0);
            fprintf(stderr, "levels: level %d: planned %d, %d pieces, %lld candidates (max %lld), work %lld (max %lld), entries %llu + total vs cap %llu, keys %llu vs table %llu\n",
                    S.next_cost, (int)planned, np, (long long)total, (long long)P.max_total, (long long)(total * P.sp.R),
                    (long long)P.max_work, (unsigned long long)S.n_entries, (unsigned long long)P.entry_cap,
                    (unsigned long long)S.keys_upper, (unsigned long long)P.table_cap);
        }
    }
    h->stats[LTL_K_LEVELS].units += S.offered - h->offered;
    h->stats[LTL_K_LEVELS].bytes += S.alg_bytes;
    u64 admitted_run = h->admitted;
    for (int k = 0; k < S.n_rows; k++) {
        const LevelRow& r = S.rows[k];
        if (r.cost == P.nostore_cost) {  // (what ltl_core_run_search does on entering the last level)
            h->store_results = false;
            h->unstored_from = S.unstored_from;
        }
        bucket[(size_t)r.cost] = std::make_pair((i64)r.first_entry, (i64)r.end_entry);
        known[(size_t)r.cost] = 1;
        admitted_run += r.admitted;
        ltl_level_stats& row = rows[(*n_rows)++];
        row.cost = r.cost;
        row.status = r.status;
        row.offered = r.offered;
        row.admitted = r.admitted;
        row.duplicates = r.duplicates;
        row.bytes = admitted_run * h->entry_bytes;  // reference _speedups.pyx:260
        row.first_entry = r.first_entry;
        row.end_entry = r.end_entry;
        row.ms = ms / (double)S.n_rows;
    }
    h->n_entries = S.n_entries;
    h->offered = S.offered;
    h->admitted = S.admitted;
    h->duplicates = S.duplicates;
    h->keys_upper = S.keys_upper;
    *next_cost = S.next_cost;
    if (S.status == LTL_S_SOLVED) {
        *status = LTL_S_SOLVED;
        *op = S.sol_op;
        *li = S.sol_li;
        *ri = S.sol_ri;
        h->pending_purge = S.sol_gbase + S.sol_cut;  // keys filed at or above the cut are not members (run_chunk)
        if (S.pend_count > 0 && h->store_results) {  // admitted, records written; matrices only if somebody asks for them
            PendingMat pm;
            pm.n_base = S.pend_base;
            pm.count = S.pend_count;
            h->pending_mat.push_back(std::move(pm));
        }
    }
    return LTL_OK;
}

// The whole cost-level loop in one call (include/ltl_core.h).  Host work per level is a handful of integer operations
// here instead of a trip through the caller's interpreter: searches of small levels are bound by exactly that.
int ltl_core_run_search(ltl_core* h, const int32_t op_cost[8], uint32_t op_mask, const int64_t* bucket_cost,
                        const int64_t* bucket_first, const int64_t* bucket_end, int n_buckets, int first_cost, int ceiling,
                        int store_last_level, ltl_level_stats* rows, int max_rows, int* n_rows, int* status, int* op,
                        int64_t* li, int64_t* ri, int* end_cost) {
    ENTER(h);
    if (!op_cost || (n_buckets && (!bucket_cost || !bucket_first || !bucket_end)) || n_buckets < 0 || !n_rows || !status || !op ||
        !li || !ri || !end_cost || (max_rows && !rows) || max_rows < 0)
        return h->fail(LTL_ERR_ARG, "null argument");
    *n_rows = 0;
    *status = LTL_S_DONE;
    *op = -1;
    *li = *ri = -1;
    *end_cost = first_cost;
    // connective order of a level: reference formula.py:24
    static const int ORDER[7] = {OP_NOT, OP_AND, OP_OR, OP_NEXT, OP_FINALLY, OP_GLOBALLY, OP_UNTIL};
    for (int k = 1; k < 8; k++)
        if (((op_mask >> k) & 1u) && op_cost[k] < 1) return h->fail(LTL_ERR_ARG, "connective costs must be positive");
    if (ceiling - first_cost > max_rows) return h->fail(LTL_ERR_ARG, "run_search: fewer stats rows than cost levels");
    std::vector<std::pair<i64, i64>> bucket((size_t)std::max(ceiling, 1), std::make_pair((i64)0, (i64)0));  // by cost
    std::vector<char> known((size_t)std::max(ceiling, 1), 0);
    for (int b = 0; b < n_buckets; b++) {
        if (bucket_cost[b] < 0 || bucket_first[b] < 0 || bucket_end[b] < bucket_first[b] || (u64)bucket_end[b] > h->n_entries)
            return h->fail(LTL_ERR_ARG, "run_search: bucket outside the store");
        if (bucket_cost[b] < ceiling) {
            bucket[(size_t)bucket_cost[b]] = std::make_pair((i64)bucket_first[b], (i64)bucket_end[b]);
            known[(size_t)bucket_cost[b]] = 1;
        }
    }
    std::vector<ltl_segment> segs;
    std::vector<Unit> units;
    int c_start = first_cost;
    {   // the small levels a search starts with: one launch (levels.cuh)
        int rc = run_levels_device(h, op_cost, op_mask, bucket, known, first_cost, ceiling, store_last_level, rows, n_rows, status, op,
                                   li, ri, &c_start);
        if (rc) return rc;
        *end_cost = std::min(c_start, ceiling);
        if (*status == LTL_S_SOLVED || *status == LTL_S_TIMEOUT) return LTL_OK;
    }
    for (int c = c_start; c < ceiling; c++) {
        *end_cost = c;
        const auto t0 = std::chrono::steady_clock::now();
        // begin_level: reference cache.py:144-152
        const u64 n0 = h->n_entries, o0 = h->offered, a0 = h->admitted, d0 = h->duplicates;
        if (c == ceiling - 1 && !store_last_level && h->unstored_from == ~0ull) h->store_results = false;
        // the level's segments: child-cost pairing of reference enumerator.py:254-268, dispatch order of 271-296
        segs.clear();
        for (int oi = 0; oi < 7; oi++) {
            const int o = ORDER[oi];
            if (!((op_mask >> o) & 1u)) continue;
            const int w = op_cost[o];
            const bool unary = o == OP_NOT || o == OP_NEXT || o == OP_FINALLY || o == OP_GLOBALLY;
            if (unary) {
                const int a = c - w;
                if (a >= 1 && bucket[(size_t)a].second > bucket[(size_t)a].first)
                    segs.push_back(ltl_segment{o, 0, bucket[(size_t)a].first, bucket[(size_t)a].second, -1, -1});
                continue;
            }
            const bool commutative = o == OP_AND || o == OP_OR;
            for (int a = 1; a < c - w; a++) {
                const int b = c - w - a;
                if (b < 1) continue;
                if (commutative && a > b) break;
                const auto& A = bucket[(size_t)a];
                const auto& B = bucket[(size_t)b];
                if (A.second == A.first || B.second == B.first) continue;
                segs.push_back(ltl_segment{o, commutative && a == b ? 1 : 0, A.first, A.second, B.first, B.second});
            }
        }
        units.clear();
        int rc = expand_segments(h, segs.data(), (int)segs.size(), units);
        if (rc) return rc;
        int seg_index = -1;
        rc = run_units(h, units, true, status, &seg_index, li, ri);
        if (rc) return rc;
        if (*status == LTL_S_OOM || *status == LTL_S_TIMEOUT) return LTL_OK;  // no row for a level that did not end (enumerator.py:243-245)
        // end_level: reference cache.py:154-166
        // (a bucket that exists already -- negated atoms of the NNF fragment can cost as much as this level -- grows)
        bucket[(size_t)c] = std::make_pair(known[(size_t)c] ? bucket[(size_t)c].first : (i64)n0, (i64)h->n_entries);
        known[(size_t)c] = 1;
        ltl_level_stats& row = rows[(*n_rows)++];
        row.cost = c;
        row.status = *status;
        row.offered = h->offered - o0;
        row.admitted = h->admitted - a0;
        row.duplicates = h->duplicates - d0;
        row.bytes = h->admitted * h->entry_bytes;  // reference _speedups.pyx:260
        row.first_entry = (int64_t)bucket[(size_t)c].first;
        row.end_entry = (int64_t)bucket[(size_t)c].second;
        row.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (*status == LTL_S_SOLVED) {
            *op = seg_index >= 0 ? segs[(size_t)seg_index].op : -1;
            return LTL_OK;
        }
    }
    *end_cost = ceiling;
    return LTL_OK;
}

int ltl_core_screen_unary(ltl_core* h, int op, int64_t c0, int64_t c1, int* status, int64_t* li, int64_t* ri) {
    ltl_segment s{op, 0, c0, c1, -1, -1};
    int seg;
    return ltl_core_run_level(h, &s, 1, status, &seg, li, ri);
}

int ltl_core_screen_binary(ltl_core* h, int op, int64_t a0, int64_t a1, int64_t b0, int64_t b1, int tri, int* status,
                           int64_t* li, int64_t* ri) {
    ltl_segment s{op, tri ? 1 : 0, a0, a1, b0, b1};
    int seg;
    return ltl_core_run_level(h, &s, 1, status, &seg, li, ri);
}

int ltl_core_contains(ltl_core* h, const uint64_t* cm, int* found) {
    ENTER(h);
    if (!cm || !found) return h->fail(LTL_ERR_ARG, "null argument");
    const i64 e = (i64)h->n_entries;  // staged past the end of the store, never admitted
    int rc;
    if ((rc = stage_matrix(h, cm, e))) return rc;
    ChunkOut co;
    if ((rc = single_chunk(h, e, MODE_LOOKUP, &co))) return rc;
    *found = h->h_ctl->found ? 1 : 0;
    return LTL_OK;
}

int ltl_core_fingerprint_of(ltl_core* h, const uint64_t* cm, uint64_t* hi, uint64_t* lo) {
    ENTER(h);
    if (!cm || !hi || !lo) return h->fail(LTL_ERR_ARG, "null argument");
    const i64 e = (i64)h->n_entries;
    int rc;
    if ((rc = stage_matrix(h, cm, e))) return rc;
    ChunkOut co;
    if ((rc = single_chunk(h, e, MODE_FP_ONLY, &co))) return rc;
    *hi = h->h_ctl->fp_hi;
    *lo = h->h_ctl->fp_lo;
    return LTL_OK;
}

int ltl_core_entry_fingerprints(ltl_core* h, int64_t first, int64_t count, uint64_t* hi, uint64_t* lo) {
    ENTER(h);
    if (first < 0 || count < 0 || (u64)(first + count) > h->n_entries) return h->fail(LTL_ERR_ARG, "entry range outside the store");
    if (count == 0) return LTL_OK;
    if (!hi || !lo) return h->fail(LTL_ERR_ARG, "null argument");
    if ((u64)(first + count) > h->unstored_from) return h->fail(LTL_ERR_ARG, "matrices of these entries were not stored");
    {
        int rcf = flush_materialize(h);
        if (rcf) return rcf;
    }
    std::vector<u64> host;
    for (i64 done = 0; done < count;) {
        const i64 take = std::min<i64>(count - done, 1 << 20);
        if (take > h->fp_cap) {
            CK(cudaStreamSynchronize(h->stream));
            cudaFree(h->d_fp);
            h->d_fp = nullptr;
            h->fp_cap = 0;
            CK(cudaMalloc(&h->d_fp, (size_t)take * 16));
            h->fp_cap = take;
        }
        std::vector<Piece> pieces;
        i64 total = 0, tiles = 0;
        Unit u{PIECE_UNARY, OP_IDENT, 0, first + done, first + done + take, -1, -1};
        push_piece(h, pieces, total, tiles, u, u.i0, u.i1, -1, -1, PIECE_UNARY);
        ChunkOut co;
        int rc = run_chunk(h, pieces, total, tiles, MODE_FP_ONLY, false, false, &co);
        if (rc) return rc;
        host.resize((size_t)take * 2);
        CK(cudaMemcpy(host.data(), h->d_fp, (size_t)take * 16, cudaMemcpyDeviceToHost));
        for (i64 k = 0; k < take; k++) {
            hi[done + k] = host[2 * k];
            lo[done + k] = host[2 * k + 1];
        }
        done += take;
    }
    return LTL_OK;
}

int ltl_core_export_cms(ltl_core* h, int64_t first, int64_t count, uint64_t* cms_out) {
    ENTER(h);
    if (first < 0 || count < 0 || (u64)(first + count) > h->n_entries) return h->fail(LTL_ERR_ARG, "entry range outside the store");
    if (count == 0) return LTL_OK;
    if (!cms_out) return h->fail(LTL_ERR_ARG, "null argument");
    if ((u64)(first + count) > h->unstored_from) return h->fail(LTL_ERR_ARG, "matrices of these entries were not stored");
    {
        int rcf = flush_materialize(h);
        if (rcf) return rcf;
    }
    const i64 max_batch = std::max<i64>(1, ((i64)256 << 20) / (h->n * 8));
    u64* d_out = nullptr;
    const i64 batch = std::min<i64>(count, max_batch);
    CK(cudaMalloc(&d_out, (size_t)batch * h->n * 8));
    for (i64 done = 0; done < count;) {
        const i64 take = std::min<i64>(batch, count - done);
        const i64 f = first + done;
        const i64 groups = ((f + take + 31) >> 5) - (f >> 5);
        const i64 threads = groups * h->n * 32;
        {
            ScopedTimer t(h, LTL_K_MISC, (u64)take, 16.0 * (double)h->n * (double)take);
            k_export<<<(unsigned)((threads + 255) / 256), 256, 0, h->stream>>>((const u64*)h->cms.base, f, take, h->n, d_out);
        }
        void* host_dst = cms_out + (size_t)done * h->n_api;
        std::vector<u64> packed;
        if (h->pair) {
            packed.resize((size_t)take * h->n);
            host_dst = packed.data();
        }
        cudaError_t e = cudaMemcpyAsync(host_dst, d_out, (size_t)take * h->n * 8, cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            cudaFree(d_out);
            return h->cuda_fail(e, "export_cms");
        }
        if (h->pair)
            for (i64 k = 0; k < take; k++) unpack_pairs(packed.data() + (size_t)k * h->n, h->R_api, cms_out + (size_t)(done + k) * h->n_api);
        h->d2h_bytes += (size_t)take * h->n * 8;
        done += take;
    }
    cudaFree(d_out);
    drain_events(h);
    return LTL_OK;
}

int ltl_core_get_cm(ltl_core* h, int64_t idx, uint64_t* out) {
    if (!h) return LTL_ERR_ARG;
    if (idx < 0 || (u64)idx >= h->n_entries) return h->fail(LTL_ERR_ARG, "entry index out of range");
    return ltl_core_export_cms(h, idx, 1, out);
}

int ltl_core_export_records(ltl_core* h, int64_t first, int64_t count, int8_t* op, int32_t* lhs, int32_t* rhs) {
    ENTER(h);
    if (first < 0 || count < 0 || (u64)(first + count) > h->n_entries) return h->fail(LTL_ERR_ARG, "entry range outside the store");
    if (count == 0) return LTL_OK;
    if (!op || !lhs || !rhs) return h->fail(LTL_ERR_ARG, "null argument");
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(op, h->rec_op.base + first, (size_t)count, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lhs, h->rec_lhs.base + first * 4, (size_t)count * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rhs, h->rec_rhs.base + first * 4, (size_t)count * 4, cudaMemcpyDeviceToHost));
    h->d2h_bytes += (size_t)count * 9;
    return LTL_OK;
}

int ltl_core_get_subtree(ltl_core* h, int64_t idx, int cap, int32_t* nodes, int* n_nodes) {
    ENTER(h);
    if (!nodes || !n_nodes || cap < 1) return h->fail(LTL_ERR_ARG, "null argument");
    *n_nodes = 0;
    if (idx < 0 || (u64)idx >= h->n_entries) return h->fail(LTL_ERR_ARG, "entry index out of range");
    cap = std::min(cap, LTL_SUBTREE_MAX);
    if (!h->d_subtree) CK(cudaMalloc(&h->d_subtree, (size_t)(4 * LTL_SUBTREE_MAX + 1) * sizeof(int)));
    {
        ScopedTimer t(h, LTL_K_MISC, 1, 9.0 * cap);
        k_subtree<<<1, 1, 0, h->stream>>>((const unsigned char*)h->rec_op.base, (const int*)h->rec_lhs.base, (const int*)h->rec_rhs.base,
                                          (i64)idx, (i64)h->n_entries, cap, h->d_subtree + 1, h->d_subtree);
    }
    CK(cudaGetLastError());
    // (count and nodes in one copy: the count sits in front of the node list)
    std::vector<int> host((size_t)4 * cap + 1);
    CK(cudaMemcpyAsync(host.data(), h->d_subtree, host.size() * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->d2h_bytes += host.size() * sizeof(int);
    drain_events(h);
    if (host[0] < 0) return h->fail(LTL_ERR_ARG, "get_subtree: the formula has more nodes than the buffer");
    *n_nodes = host[0];
    memcpy(nodes, host.data() + 1, (size_t)host[0] * 4 * sizeof(int));
    return LTL_OK;
}

int ltl_core_get_record(ltl_core* h, int64_t idx, int* op, int* lhs, int* rhs) {
    if (!h) return LTL_ERR_ARG;
    if (idx < 0 || (u64)idx >= h->n_entries) return h->fail(LTL_ERR_ARG, "entry index out of range");
    int8_t o;
    int32_t l, r;
    int rc = ltl_core_export_records(h, idx, 1, &o, &l, &r);
    if (rc) return rc;
    *op = o;
    *lhs = l;
    *rhs = r;
    return LTL_OK;
}

int ltl_core_counters(ltl_core* h, uint64_t out[5]) {
    if (!h || !out) return LTL_ERR_ARG;
    out[0] = h->n_entries;
    out[1] = h->admitted * h->entry_bytes;  // reference _speedups.pyx:260
    out[2] = h->offered;
    out[3] = h->admitted;
    out[4] = h->duplicates;
    return LTL_OK;
}

int ltl_core_set_option(ltl_core* h, const char* name, int64_t value) {
    if (!h || !name) return LTL_ERR_ARG;
    if (!strcmp(name, "chunk_candidates")) {
        if (value < 1 || value > ((int64_t)1 << 30)) return h->fail(LTL_ERR_ARG, "chunk_candidates outside [1, 2^30]");
        h->chunk_cap = value;
    } else if (!strcmp(name, "deadline_ms")) {
        h->deadline_at = value > 0 ? steady_seconds() + (double)value * 1e-3 : 0.0;
    } else if (!strcmp(name, "sub_tiles")) {
        h->sub_tiles = std::max<int64_t>(LTL_WARPS_PER_CTA, value);
    } else if (!strcmp(name, "store_results")) {
        if (value && h->unstored_from != ~0ull) return h->fail(LTL_ERR_ARG, "matrices were already skipped: storing cannot resume");
        h->store_results = value != 0;
    } else if (!strcmp(name, "tiled_materialize")) {
        h->tiled_materialize = (int)value;
    } else if (!strcmp(name, "fuse_unary")) {
        h->fuse_unary = value != 0;
    } else if (!strcmp(name, "fuse_not")) {
        h->fuse_not = value != 0;
    } else if (!strcmp(name, "gate_store")) {
        h->gate_store = value != 0;
    } else if (!strcmp(name, "debug_masks")) {
        h->debug_masks = value != 0;
    } else if (!strcmp(name, "exchange_parts")) {
        h->exchange_parts = (int)std::max<int64_t>(1, std::min<int64_t>(8, value));
    } else if (!strcmp(name, "order_mat")) {
        h->order_mat = value != 0;
    } else if (!strcmp(name, "order_min")) {
        h->order_min = value;
    } else if (!strcmp(name, "order_block_bytes")) {
        h->order_block_bytes = std::max<int64_t>(1, value);
    } else if (!strcmp(name, "small_screen")) {
        h->small_screen = value != 0;
    } else if (!strcmp(name, "small_admit")) {
        h->small_admit = value != 0;
    } else if (!strcmp(name, "device_levels")) {
        h->device_levels = value != 0;
    } else if (!strcmp(name, "levels_ctas")) {
        if (value != 1 && value != 2 && value != 4 && value != 8) return h->fail(LTL_ERR_ARG, "levels_ctas must be 1, 2, 4 or 8");
        h->levels_ctas = (int)value;
    } else if (!strcmp(name, "levels_max_work")) {
        h->levels_max_work = std::max<int64_t>(0, value);
    } else if (!strcmp(name, "fuse_not_min")) {
        h->fuse_not_min = value;
    } else if (!strcmp(name, "profile")) {
        h->profile = value != 0;
    } else if (!strcmp(name, "max_split")) {
        h->max_split = (int)std::max<int64_t>(1, value);
    } else if (!strcmp(name, "force_split")) {
        h->force_split = (int)std::max<int64_t>(0, value);
    } else {
        return h->fail(LTL_ERR_ARG, std::string("unknown option ") + name);
    }
    return LTL_OK;
}

int ltl_core_kernel_stats(ltl_core* h, int cls, uint64_t* launches, double* ms, double* alg_bytes, uint64_t* units) {
    ENTER(h);
    if (cls < 0 || cls >= LTL_K_COUNT) return h->fail(LTL_ERR_ARG, "kernel class out of range");
    CK(cudaStreamSynchronize(h->stream));
    drain_events(h);
    if (launches) *launches = h->stats[cls].launches;
    if (ms) *ms = h->stats[cls].ms;
    if (alg_bytes) *alg_bytes = h->stats[cls].bytes;
    if (units) *units = h->stats[cls].units;
    return LTL_OK;
}

int ltl_core_reset_kernel_stats(ltl_core* h) {
    ENTER(h);
    CK(cudaStreamSynchronize(h->stream));
    drain_events(h);
    for (auto& s : h->stats) s = KStat();
    return LTL_OK;
}

int ltl_core_stream(ltl_core* h, void** stream_out) {
    if (!h || !stream_out) return LTL_ERR_ARG;
    *stream_out = (void*)h->stream;
    return LTL_OK;
}

// ---- multi-GPU stages ---------------------------------------------------------------------------

int ltl_core_level_size(ltl_core* h, const ltl_segment* segs, int n_segs, int64_t* total) {
    ENTER(h);
    if (!total || n_segs < 0 || (n_segs && !segs)) return h->fail(LTL_ERR_ARG, "null argument");
    std::vector<Unit> units;
    int rc = expand_segments(h, segs, n_segs, units);
    if (rc) return rc;
    i64 t = 0;
    for (auto& u : units) t += unit_count(u);
    *total = t;
    return LTL_OK;
}

int ltl_plan_level(const int32_t op_cost[8], uint32_t op_mask, const int64_t* bucket_cost, const int64_t* bucket_first,
                   const int64_t* bucket_end, int n_buckets, int cost, int cap, int32_t* op_out, int32_t* kind_out,
                   int64_t* range_out, int64_t* count_out, int* n_pieces, int64_t* total) {
    if (!op_cost || n_buckets < 0 || (n_buckets && (!bucket_cost || !bucket_first || !bucket_end)) || cap < 0 || !n_pieces || !total ||
        (cap && (!op_out || !kind_out || !range_out || !count_out)) || cost < 1 || cost > LTL_LV_MAX_COST)
        return LTL_ERR_ARG;
    i64 bf[LTL_LV_MAX_COST] = {0}, be[LTL_LV_MAX_COST] = {0};
    for (int b = 0; b < n_buckets; b++)
        if (bucket_cost[b] >= 0 && bucket_cost[b] < LTL_LV_MAX_COST) {
            bf[bucket_cost[b]] = bucket_first[b];
            be[bucket_cost[b]] = bucket_end[b];
        }
    std::vector<Piece> pieces((size_t)std::max(cap, 1));
    int oc[8];
    for (int k = 0; k < 8; k++) oc[k] = op_cost[k];
    int np = 0;
    i64 tot = 0;
    double bytes = 0;
    if (!lv_plan(cost, oc, op_mask, bf, be, pieces.data(), cap, &np, &tot, &bytes, 0.0)) return LTL_ERR_ARG;
    for (int k = 0; k < np; k++) {
        op_out[k] = pieces[(size_t)k].op;
        kind_out[k] = pieces[(size_t)k].kind;
        range_out[4 * k] = pieces[(size_t)k].i0;
        range_out[4 * k + 1] = pieces[(size_t)k].i1;
        range_out[4 * k + 2] = pieces[(size_t)k].j0;
        range_out[4 * k + 3] = pieces[(size_t)k].j1;
        count_out[k] = pieces[(size_t)k].count;
    }
    *n_pieces = np;
    *total = tot;
    return LTL_OK;
}

int ltl_core_set_row_shard(ltl_core* h, int64_t word_base, int64_t total_words, ltl_exchange_fn fn, void* ctx) {
    ENTER(h);
    if (h->n_entries || h->offered) return h->fail(LTL_ERR_ARG, "set_row_shard: the core is already in use");
    // a fingerprint block is 64 STORED words: 64 API words, or 128 rows of the half-width store
    const i64 blk_words = h->pair ? 128 : 64;
    if (!fn || word_base < 0 || (word_base % blk_words) || total_words < word_base + h->n_api)
        return h->fail(LTL_ERR_ARG, "set_row_shard: word_base must be a multiple of the fingerprint block (64 words; 128 rows for "
                                    "the half-width store) and the shard must lie inside the matrix");
    if (word_base + h->n_api < total_words && (h->n_api % blk_words))
        return h->fail(LTL_ERR_ARG, "set_row_shard: only the last shard may end inside a fingerprint block");
    if (h->variant != VAR_MUELLER && h->variant != VAR_NH)
        return h->fail(LTL_ERR_ARG, "set_row_shard: needs a block-combinable fingerprint (mueller / nh)");
    h->blk_base = (u32)(word_base / blk_words);
    h->exchange = fn;
    h->exchange_ctx = ctx;
    // the budget counts whole matrices, like the reference's (reference _speedups.pyx:100, 252-253)
    h->entry_bytes = (u64)total_words * 8 + 16;
    h->cap_entries = std::min<u64>(h->cap_entries, h->budget / h->entry_bytes);
    return LTL_OK;
}

int ltl_core_set_table_shard(ltl_core* h, int shard, int n_shards) {
    ENTER(h);
    if (!h->exchange) return h->fail(LTL_ERR_ARG, "set_table_shard: call ltl_core_set_row_shard first");
    if (h->n_entries || h->offered) return h->fail(LTL_ERR_ARG, "set_table_shard: the core is already in use");
    if (n_shards < 1 || n_shards > LTL_MAX_WORLD || shard < 0 || shard >= n_shards) return h->fail(LTL_ERR_ARG, "set_table_shard: bad shard");
    h->table_shard = shard;
    h->table_shards = n_shards;
    return LTL_OK;
}

int ltl_core_stage_eval(ltl_core* h, const ltl_segment* segs, int n_segs, int64_t lo, int64_t hi, uint64_t* d_fp,
                        int64_t* solver_rank) {
    ENTER(h);
    if (!solver_rank || n_segs < 0 || (n_segs && !segs)) return h->fail(LTL_ERR_ARG, "null argument");
    *solver_rank = -1;
    std::vector<Unit> units;
    int rc = expand_segments(h, segs, n_segs, units);
    if (rc) return rc;
    i64 level_total = 0;
    for (auto& u : units) level_total += unit_count(u);
    if (lo < 0 || hi < lo || hi > level_total) return h->fail(LTL_ERR_ARG, "rank range outside the level");
    if (hi == lo) return LTL_OK;
    if (!d_fp) return h->fail(LTL_ERR_ARG, "null fingerprint buffer");
    if ((rc = flush_materialize(h))) return rc;
    std::vector<Piece> pieces;
    const i64 cap = std::min<i64>(h->chunk_cap, (i64)1 << 26);
    for (i64 c0 = lo; c0 < hi; c0 += cap) {
        const i64 c1 = std::min<i64>(hi, c0 + cap);
        pieces.clear();
        i64 total = 0, tiles = 0;
        plan_range(h, units, c0, c1, pieces, total, tiles);
        if (total != c1 - c0) return h->fail(LTL_ERR_CUDA, "internal: range plan does not cover the slice");
        h->fp_ext = (u64*)d_fp + 2 * (c0 - lo);
        ChunkOut co;
        rc = run_chunk(h, pieces, total, tiles, MODE_FP_ONLY, true, false, &co);
        h->fp_ext = nullptr;
        if (rc) return rc;
        if (h->h_ctl->solver_c != ~0ull) {
            *solver_rank = c0 + (i64)h->h_ctl->solver_c;
            break;  // fingerprints above a solver are never used
        }
    }
    return LTL_OK;
}

int ltl_core_stage_file(ltl_core* h, const uint64_t* d_tuples, int64_t count, unsigned char* d_win, int64_t* n_win) {
    ENTER(h);
    if (count < 0 || !n_win) return h->fail(LTL_ERR_ARG, "bad argument");
    *n_win = 0;
    if (count == 0) return LTL_OK;
    if (!d_tuples || !d_win) return h->fail(LTL_ERR_ARG, "null argument");
    int rc;
    if ((rc = apply_purge(h))) return rc;
    if ((rc = ensure_table(h, h->keys_upper + (u64)count))) return rc;
    if ((rc = ensure_scratch(h, count))) return rc;
    CK(cudaMemsetAsync(&h->d_ctl->total, 0, sizeof(u64), h->stream));
    const unsigned nb = (unsigned)((count + 255) / 256);
    {
        ScopedTimer t(h, LTL_K_RESOLVE, (u64)count, (double)count * 56.0);
        k_file_insert<<<nb, 256, 0, h->stream>>>((const u64*)d_tuples, (u64)count, h->table, h->table_cap - 1, h->offered, h->d_slot);
        k_file_verdict<<<nb, 256, 0, h->stream>>>((const u64*)d_tuples, h->d_slot, (u64)count, h->table, d_win, h->d_ctl);
        h->stats[LTL_K_RESOLVE].launches += 1;  // (two kernels under one timer)
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->d2h_bytes += sizeof(Ctl);
    drain_events(h);
    *n_win = (int64_t)h->h_ctl->total;
    h->keys_upper += h->h_ctl->total;
    return LTL_OK;
}

int ltl_core_stage_route(ltl_core* h, const uint64_t* d_fp, int64_t count, uint64_t rank_base, int world, uint64_t* d_send,
                         int64_t* counts_out) {
    ENTER(h);
    if (count < 0 || world < 1 || world > LTL_MAX_WORLD || !counts_out) return h->fail(LTL_ERR_ARG, "stage_route: bad argument");
    for (int d = 0; d < world; d++) counts_out[d] = 0;
    if (count == 0) return LTL_OK;
    if (!d_fp || !d_send) return h->fail(LTL_ERR_ARG, "null argument");
    const u32 nb = (u32)((count + 1023) / 1024);
    const size_t cells = (size_t)world * nb;
    if (cells + 1 > h->route_cap) {
        CK(cudaStreamSynchronize(h->stream));
        cudaFree(h->d_route_hist);
        cudaFree(h->d_route_off);
        h->d_route_hist = h->d_route_off = nullptr;
        h->route_cap = 0;
        const size_t cap = std::max<size_t>(cells + 1, 1 << 14);
        CK(cudaMalloc(&h->d_route_hist, cap * 4));
        CK(cudaMalloc(&h->d_route_off, cap * 4));
        h->route_cap = cap;
    }
    {
        ScopedTimer t(h, LTL_K_MISC, (u64)count, (double)count * 56.0);
        k_route_count<<<nb, 1024, 0, h->stream>>>((const u64*)d_fp, (u64)count, world, h->d_route_hist, nb);
        k_plan_scan<<<1, 1024, 0, h->stream>>>(h->d_route_hist, (int)cells, h->d_route_off);
        k_route_scatter<<<nb, 1024, 0, h->stream>>>((const u64*)d_fp, (u64)count, world, rank_base, h->d_route_off, nb, (u64*)d_send);
        h->stats[LTL_K_MISC].launches += 2;  // (three kernels under one timer)
    }
    CK(cudaGetLastError());
    u32 bounds[LTL_MAX_WORLD + 1];
    CK(cudaMemcpy2DAsync(bounds, 4, h->d_route_off, (size_t)nb * 4, 4, (size_t)world + 1, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->d2h_bytes += 4 * (size_t)(world + 1);
    drain_events(h);
    for (int d = 0; d < world; d++) counts_out[d] = (int64_t)(bounds[d + 1] - bounds[d]);
    return LTL_OK;
}

int ltl_core_stage_winners(ltl_core* h, const uint64_t* d_tuples, const unsigned char* d_win, int64_t count, uint64_t rank_base,
                           int64_t level_lo, int64_t* d_out, int64_t* n_out) {
    ENTER(h);
    if (count < 0 || !n_out) return h->fail(LTL_ERR_ARG, "stage_winners: bad argument");
    *n_out = 0;
    if (count == 0) return LTL_OK;
    if (!d_tuples || !d_win || !d_out) return h->fail(LTL_ERR_ARG, "null argument");
    int rc;
    if ((rc = ensure_scratch(h, count))) return rc;
    const unsigned nb = (unsigned)((count + RES_CTA - 1) / RES_CTA);
    CK(cudaMemsetAsync(h->d_flagw, 0, (size_t)nb * (RES_CTA / 32) * 4, h->stream));
    {
        ScopedTimer t(h, LTL_K_MISC, (u64)count, (double)count * 33.0);
        k_win_flags<<<(unsigned)((count + 255) / 256), 256, 0, h->stream>>>((const u64*)d_tuples, d_win, (u64)count, rank_base, h->d_flagw);
        k_flag_count<<<nb, RES_CTA, 0, h->stream>>>(h->d_flagw, (u64)count, h->d_blocksum);
        k_scan<<<1, 1024, 0, h->stream>>>(h->d_blocksum, nb, h->d_blockoff, h->d_ctl);
        k_emit_ranks<<<nb, RES_CTA, 0, h->stream>>>(h->d_flagw, h->d_blockoff, (u64)count, (i64)level_lo, (i64*)d_out);
        h->stats[LTL_K_MISC].launches += 3;  // (four kernels under one timer)
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->d2h_bytes += sizeof(Ctl);
    drain_events(h);
    *n_out = (int64_t)h->h_ctl->total;
    return LTL_OK;
}

int ltl_core_stage_decode(ltl_core* h, const ltl_segment* segs, int n_segs, const int64_t* d_ranks, int64_t count,
                          unsigned char* d_op, int32_t* d_lhs, int32_t* d_rhs) {
    ENTER(h);
    if (count < 0) return h->fail(LTL_ERR_ARG, "bad argument");
    if (count == 0) return LTL_OK;
    if (!d_ranks || !d_op || !d_lhs || !d_rhs) return h->fail(LTL_ERR_ARG, "null argument");
    std::vector<Unit> units;
    int rc = expand_segments(h, segs, n_segs, units);
    if (rc) return rc;
    i64 level_total = 0;
    for (auto& u : units) level_total += unit_count(u);
    std::vector<Piece> pieces;
    i64 total = 0, tiles = 0;
    plan_range(h, units, 0, level_total, pieces, total, tiles);
    if ((rc = ensure_pieces(h, (int)pieces.size()))) return rc;
    CK(cudaStreamSynchronize(h->stream));
    memcpy(h->h_pieces, pieces.data(), sizeof(Piece) * pieces.size());
    CK(cudaMemcpyAsync(h->d_pieces, h->h_pieces, sizeof(Piece) * pieces.size(), cudaMemcpyHostToDevice, h->stream));
    {
        ScopedTimer t(h, LTL_K_EMIT, (u64)count, (double)count * 17.0);
        k_decode<<<(unsigned)((count + 255) / 256), 256, 0, h->stream>>>((const i64*)d_ranks, (u64)count, h->d_pieces,
                                                                          (int)pieces.size(), d_op, d_lhs, d_rhs);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    drain_events(h);
    return LTL_OK;
}

int ltl_core_stage_append(ltl_core* h, const unsigned char* d_op, const int32_t* d_lhs, const int32_t* d_rhs, int64_t count,
                          uint64_t offered_delta, uint64_t duplicates_delta) {
    ENTER(h);
    if (count < 0) return h->fail(LTL_ERR_ARG, "bad argument");
    if (count > 0) {
        if (!d_op || !d_lhs || !d_rhs) return h->fail(LTL_ERR_ARG, "null argument");
        if (h->n_entries + (u64)count > h->cap_entries) return h->fail(LTL_ERR_BUDGET, "append beyond the entry capacity");
        int rc = ensure_records(h, h->n_entries + (u64)count);
        if (rc) return rc;
        CK(cudaMemcpyAsync(h->rec_op.base + h->n_entries, d_op, (size_t)count, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(h->rec_lhs.base + h->n_entries * 4, d_lhs, (size_t)count * 4, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(h->rec_rhs.base + h->n_entries * 4, d_rhs, (size_t)count * 4, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (h->store_results) {
            PendingMat pm;
            pm.n_base = h->n_entries;
            pm.count = (u64)count;
            h->pending_mat.push_back(std::move(pm));
        }
        else if (h->unstored_from == ~0ull) h->unstored_from = h->n_entries;
        h->n_entries += (u64)count;
        h->admitted += (u64)count;
    }
    h->offered += offered_delta;
    h->duplicates += duplicates_delta;
    return LTL_OK;
}

int ltl_core_stage_purge(ltl_core* h, uint64_t global_rank_cut) {
    ENTER(h);
    ScopedTimer t(h, LTL_K_PURGE, h->table_cap, (double)h->table_cap * sizeof(Slot));
    k_purge<<<(unsigned)((h->table_cap + 255) / 256), 256, 0, h->stream>>>(h->table, h->table_cap, global_rank_cut);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    return LTL_OK;
}

uint64_t ltl_pool_trim(void) { return (uint64_t)pool_trim(); }

int ltl_core_host_times(ltl_core* h, double out[3]) {
    if (!h || !out) return LTL_ERR_ARG;
    out[0] = h->grow_ms;
    out[1] = h->sync_ms;
    out[2] = h->plan_ms;
    return LTL_OK;
}

int ltl_core_transfer_stats(ltl_core* h, uint64_t out[2]) {
    if (!h || !out) return LTL_ERR_ARG;
    out[0] = h->h2d_bytes;
    out[1] = h->d2h_bytes;
    return LTL_OK;
}

int ltl_core_info(ltl_core* h, uint64_t out[6]) {
    if (!h || !out) return LTL_ERR_ARG;
    out[0] = h->cap_entries;
    out[1] = h->cms.mapped;
    out[2] = h->table_cap;
    out[3] = (u64)h->chunk_cap;
    out[4] = (h->cms.vmm ? 1 : 0) | (h->device_oom ? 2 : 0) | (h->gated_skips << 8);
    out[5] = (u64)h->n_api;
    return LTL_OK;
}

}  // extern "C"
