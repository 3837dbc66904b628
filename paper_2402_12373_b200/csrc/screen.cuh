// screen.cuh -- the two hot kernels of the screening core, templated on W = words per row.
//
//   k_screen<W, KIND>      "phase A" (KIND_MUELLER / KIND_BITS), and with KIND_REWRITE the tile-shaped phase B: one warp per tile of (<= 4 entries of one operand) x (32 entries of
//       the other); every lane evaluates its candidates' characteristic matrices row by row IN REGISTERS
//       (nothing is written back), counts P/N classification errors (fused solve check, reference
//       _speedups.pyx:327-333), folds the rows into the 126-bit fingerprint (reference _speedups.pyx:185-231)
//       and files the fingerprint in the uniqueness table with atomicMin(rank)
//       (= the sequential first-wins admission of _speedups.pyx:245-262, made order-independent).
//   k_materialize<W>       "phase B": one warp per 32 consecutive NEW entries; re-evaluates only the
//       winners from their (op, lhs, rhs) records and appends them to the store with full-line writes.
//
// Reference loop being replaced: _speedups.pyx:337-380 (screen_unary / screen_binary).
#pragma once
#include "semantics.cuh"

// ------------------------------------------------------------------------------------------------
// rank helpers

__host__ __device__ __forceinline__ u64 piece_rank(const Piece& pc, i64 i, i64 j) {
    if (pc.kind == PIECE_UNARY) return (u64)pc.cbase + (u64)(i - pc.i0);
    if (pc.kind == PIECE_RECT) return (u64)pc.cbase + (u64)(i - pc.i0) * (u64)(pc.j1 - pc.j0) + (u64)(j - pc.j0);
    return (u64)pc.cbase + tri_before((u64)(i - pc.i0), (u64)(pc.j1 - 1 - pc.i0)) + (u64)(j - i - 1);
}

// inverse of piece_rank: chunk-local rank -> (i, j); j = -1 for unary pieces
__host__ __device__ inline void piece_unrank(const Piece& pc, u64 c, i64* i, i64* j) {
    u64 local = c - (u64)pc.cbase;
    if (pc.kind == PIECE_UNARY) {
        *i = pc.i0 + (i64)local;
        *j = -1;
    } else if (pc.kind == PIECE_RECT) {
        u64 nj = (u64)(pc.j1 - pc.j0);
        u64 q = local / nj;
        *i = pc.i0 + (i64)q;
        *j = pc.j0 + (i64)(local - q * nj);
    } else {
        u64 m = (u64)(pc.j1 - 1 - pc.i0);
        // largest q with T(q) <= local, T(q) = q*m - q(q-1)/2
        double b = 2.0 * (double)m + 1.0;
        double disc = b * b - 8.0 * (double)local;
        if (disc < 0) disc = 0;
        i64 q = (i64)((b - sqrt(disc)) * 0.5);
        if (q < 0) q = 0;
        if ((u64)q > m) q = (i64)m;
        while (q > 0 && tri_before((u64)q, m) > local) q--;
        while (tri_before((u64)q + 1, m) <= local) q++;
        *i = pc.i0 + q;
        *j = *i + 1 + (i64)(local - tri_before((u64)q, m));
    }
}

#ifdef __CUDACC__

// mix64 for the hot loop.  With -DLTL_SHIFT_MADHI the three `hi >> s` of the xor-shifts are computed as
// multiply-high on the FMA pipe (hi * 2^(32-s) >> 32) instead of shifts on the ALU pipe (A/B switch: the loop
// is ALU-pipe bound, see profiles/README.md).
__device__ __forceinline__ u64 mix64_hot(u64 x) {
#ifdef LTL_SHIFT_MADHI
    u32 lo = (u32)x, hi = (u32)(x >> 32);
    lo ^= __funnelshift_r(lo, hi, 30);
    hi ^= __umulhi(hi, 1u << 2);
    x = (((u64)hi << 32) | lo) * K_MIX1;
    lo = (u32)x, hi = (u32)(x >> 32);
    lo ^= __funnelshift_r(lo, hi, 27);
    hi ^= __umulhi(hi, 1u << 5);
    x = (((u64)hi << 32) | lo) * K_MIX2;
    lo = (u32)x, hi = (u32)(x >> 32);
    lo ^= __funnelshift_r(lo, hi, 31);
    hi ^= __umulhi(hi, 1u << 1);
    return ((u64)hi << 32) | lo;
#else
    return mix64(x);
#endif
}

// a * b + c with a 64-bit accumulator: exactly one IMAD.WIDE.U32 (the C form made ptxas split the add)
__device__ __forceinline__ u64 mad_wide(u32 a, u32 b, u64 c) {
    u64 d;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

// ------------------------------------------------------------------------------------------------
// fingerprint finalisation + table filing for one candidate

template <bool MUELLER>  // true for both hashed variants (Mueller, NH): the two sums are finalised the same way
__device__ __forceinline__ void finish_candidate(const ScreenParams& p, u64 c, u64 s0, u64 s1, u32 err) {
    u64 hi, lo;
    if (MUELLER) {  // reference _speedups.pyx:203-204
        hi = mix64(s0) & K_HI_CLEAR;
        lo = mix64(s1);
    } else {
        hi = s0;
        lo = s1;
    }
    // reference _speedups.pyx:223-229: clear the lowest mask_k bits of the 128-bit value
    if (p.mask_k >= 64) {
        lo = 0;
        if (p.mask_k > 64) hi &= ~((1ull << (p.mask_k - 64)) - 1ull);
    } else if (p.mask_k > 0) {
        lo &= ~((1ull << p.mask_k) - 1ull);
    }
    const bool solves = p.check_solve && (int)err <= p.err_max;
    if (solves) atomicMin(&p.ctl->solver_c, c);
    if (p.mode == MODE_FP_ONLY) {
        if (p.fp_out) {
            p.fp_out[2 * c] = hi;
            p.fp_out[2 * c + 1] = lo;
        }
        if (c == 0) {
            p.ctl->fp_hi = hi;
            p.ctl->fp_lo = lo;
        }
        return;
    }
    if (p.owner_world > 1 && fp_owner(hi, lo, p.owner_world) != p.owner_rank) {  // another shard's key
        if (p.mode == MODE_LOOKUP) p.ctl->found = 0ull;
        else p.slot[c] = LTL_NONE;
        return;
    }
    if (p.mode == MODE_LOOKUP) {
        u64 s = table_find(p.table, p.table_mask, hi, lo);
        p.ctl->found = (s != ~0ull && ld_rank(p.table + s) != LTL_RANK_NONE) ? 1ull : 0ull;
        return;
    }
    if (solves) {  // a solving candidate is returned, never admitted (reference _speedups.pyx:372-374)
        p.slot[c] = LTL_NONE;
        return;
    }
    u64 s = table_find_or_claim(p.table, p.table_mask, hi, lo);
    u64 old = atomicMin(&p.table[s].rank, p.gbase + c);
    p.slot[c] = (old < p.gbase) ? LTL_NONE : (u32)s;  // key already a member from an earlier chunk
}

// ------------------------------------------------------------------------------------------------
// per-warp asynchronous staging of the lane operand: in the group layout the 32 lanes' words k, k+1, ... of
// one storage group are ONE contiguous stream of 256-byte lines, so a warp prefetches it with 1-D bulk
// copies (TMA engine, cp.async.bulk) into its private shared-memory ring, completion on an mbarrier.

#ifndef LTL_ROW_UNROLL
#define LTL_ROW_UNROLL 2
#endif
constexpr int kRowUnroll = LTL_ROW_UNROLL;

template <int W>
struct Ring {
    static constexpr int RPC = (W <= 8) ? 8 / W : 1;      // rows per stage
    static constexpr int STAGES = (W <= 8) ? 3 : 2;
    static constexpr int LANE_U64 = RPC * W * 32;          // lane operand: 64-bit words per stage (<= 2 KiB for W <= 8)
    static constexpr int ROW_U64 = 4 * RPC * W;            // row operands: up to 4 entries x the stage's words
    static constexpr int STAGE_U64 = LANE_U64 + ROW_U64;
    static constexpr int WARP_U64 = STAGES * STAGE_U64;
    static constexpr int CTA_BYTES = LTL_WARPS_PER_CTA * WARP_U64 * 8 + LTL_WARPS_PER_CTA * STAGES * 8;
    static constexpr bool CHUNK_FOLD = (64 % (RPC * W)) == 0;  // hash blocks end on stage boundaries
};

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra LAB_DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "LAB_DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 8-byte asynchronous copy (LDGSTS) whose completion is reported to an mbarrier by the issuing thread
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(u64* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// ------------------------------------------------------------------------------------------------
// one warp tile

// connective of slot t of a tile: OPS is either one opcode (every slot applies it to a different row operand)
// or >= 2 opcodes packed one nibble each (fused unary tile: every slot applies its own connective)
template <int OPS>
__host__ __device__ constexpr int slot_op(int t) {
    return OPS < 16 ? OPS : ((OPS >> (4 * t)) & 15);
}
template <int OPS, int W, bool PAIR>
__device__ __forceinline__ void apply_slot(const int t, u64 (&out)[W], const u64 (&x)[W], const u64 (&y)[W], const u64 (&m)[W]) {
    switch (t) {  // t is a constant after unrolling
        case 0: apply_row<slot_op<OPS>(0), W, PAIR>(out, x, y, m); break;
        case 1: apply_row<slot_op<OPS>(1), W, PAIR>(out, x, y, m); break;
        case 2: apply_row<slot_op<OPS>(2), W, PAIR>(out, x, y, m); break;
        default: apply_row<slot_op<OPS>(3), W, PAIR>(out, x, y, m); break;
    }
}
__host__ __device__ constexpr bool op_unary_c(int op) {
    return op == OP_IDENT || op == OP_NOT || op == OP_NEXT || op == OP_FINALLY || op == OP_GLOBALLY;
}
template <int OPS>
__host__ __device__ constexpr bool ops_need_mask() {
    return OPS < 16 ? (OPS == OP_NOT || OPS == OP_GLOBALLY)
                    : ((OPS & 15) == OP_NOT || (OPS & 15) == OP_GLOBALLY || ((OPS >> 4) & 15) == OP_NOT ||
                       ((OPS >> 4) & 15) == OP_GLOBALLY || ((OPS >> 8) & 15) == OP_NOT || ((OPS >> 8) & 15) == OP_GLOBALLY ||
                       ((OPS >> 12) & 15) == OP_NOT || ((OPS >> 12) & 15) == OP_GLOBALLY);
}

template <int W, int KIND, int OP, int TI, bool XL, bool PAIR>
__device__ __forceinline__ void tile_eval(const ScreenParams& p, const Piece& pc, const i64 row0, const i64 lg,
                                          const int split, const int lane, u64* __restrict__ sbuf, u64* bars) {
    constexpr bool MUELLER = KIND == KIND_MUELLER;
    constexpr bool NH = KIND == KIND_NH;
    constexpr bool HASHED = MUELLER || NH;
    constexpr bool REWRITE = KIND == KIND_REWRITE;
    constexpr bool FUSED = OP >= 16;
    constexpr bool BIN = !op_unary_c(slot_op<OP>(0));
    constexpr bool NEEDM = ops_need_mask<OP>();
    const i64 n = p.n;
    const i64 e = lg * 32 + lane;  // the lane operand's entry index

    const int r0 = split * p.rows_per_split;
    const int r1 = min(p.R, r0 + p.rows_per_split);

    // candidate of (lane, slot t): validity and chunk-local rank
    const bool lane_in = pc.kind == PIECE_UNARY ? (e >= pc.i0 && e < pc.i1)
                         : pc.kind == PIECE_RECT ? (pc.swap ? (e >= pc.i0 && e < pc.i1) : (e >= pc.j0 && e < pc.j1))
                                                 : (e < pc.j1);
    auto slot_rank = [&](const int t, u64* c) -> bool {
        i64 ci, cj;
        if (pc.kind == PIECE_UNARY) {
            ci = e;
            cj = -1;
        } else if (pc.kind == PIECE_RECT && pc.swap) {
            ci = e;
            cj = row0 + t;
        } else {
            ci = row0 + t;
            cj = e;
        }
        if (!(lane_in && (pc.kind != PIECE_TRI || cj > ci))) return false;
        *c = FUSED ? (u64)pc.fcbase[t] + (u64)(e - pc.i0) : piece_rank(pc, ci, cj);
        return true;
    };
    u64* __restrict__ pd[TI];  // REWRITE: where this lane's slot-t matrix goes (null: not a winner)
    if (REWRITE) {
        bool any = false;
#pragma unroll
        for (int t = 0; t < TI; t++) {
            u64 c;
            pd[t] = nullptr;
            if (slot_rank(t, &c)) {
                const u32 d = p.dest[c];
                if (d != LTL_NONE) {
                    pd[t] = p.cms_out + cm_index(p.n_base + (i64)d, n, 0);
                    any = true;
                }
            }
        }
        if (!__any_sync(0xFFFFFFFFu, any)) return;  // no winner in this tile
    }

    u64 s0[TI], s1[TI], h0[TI], h1[TI];
    // Verdict bits (MSB of word 0 of every row) are COUNTED with one multiply-add-high per row on the FMA pipe
    // (ones += hi32 * 2 >> 32); the count over the positive rows is snapshotted when the row index crosses n_pos:
    // errors = (#positives - ones_pos) + (ones - ones_pos)          (reference _speedups.pyx:327-333)
    // Half-width store (PAIR): a word holds rows 2v (high half, verdict bit 63) and 2v + 1 (low half, verdict bit 31);
    // the low rows are counted in ones2 and snapshotted where THEIR positives end (p.n_pos_lo <= p.n_pos <= p.n_pos_lo + 1).
    u32 ones[TI], ones_pos[TI], ones2[TI], ones2_pos[TI];
#pragma unroll
    for (int t = 0; t < TI; t++) {
        s0[t] = s1[t] = 0;
        h0[t] = NH ? 0ull : K_SEED0;  // NH: the block's two accumulators d_0, d_1
        h1[t] = NH ? 0ull : K_SEED1;
        ones[t] = ones_pos[t] = 0;
        ones2[t] = ones2_pos[t] = 0;
    }
    u64 tw = ((u64)p.blk_base * 64ull + (u64)r0 * W + 1ull) * K_STEP;  // (k + 1) * STEP for the next (global) word k
    int d = 0;                               // next deposit (bits fingerprints)
    if (KIND == KIND_BITS) {
        const u32 kfirst = (u32)r0 * W;
        int lo_ = 0, hi_ = p.n_dep;
        while (lo_ < hi_) {
            int mid = (lo_ + hi_) >> 1;
            if (p.deps[mid].k < kfirst) lo_ = mid + 1;
            else hi_ = mid;
        }
        d = lo_;
    }

    auto fold = [&](const u32 blk_local) {  // blocked Mueller: block 0 enters as is (== reference for n <= 64)
        const u32 blk = blk_local + p.blk_base;
        const bool first = blk == 0;
#pragma unroll
        for (int t = 0; t < TI; t++) {
            if (NH) {  // oracle fp_nh: s0 += mix64(d0 ^ u), s1 += mix64(d1 + u), u = (block + 1) * STEP
                const u64 u = (u64)(blk + 1) * K_STEP;
                s0[t] += mix64(h0[t] ^ u);
                s1[t] += mix64(h1[t] + u);
                h0[t] = h1[t] = 0;
                continue;
            }
            if (first) {
                s0[t] += h0[t];
                s1[t] += h1[t];
            } else {
                s0[t] += mix64(h0[t]);
                s1[t] += mix64(h1[t]);
            }
            h0[t] = K_SEED0;
            h1[t] = K_SEED1;
        }
    };

    auto snapshot = [&]() {
#pragma unroll
        for (int t = 0; t < TI; t++) ones_pos[t] = ones[t];
    };
    auto snapshot_lo = [&]() {
#pragma unroll
        for (int t = 0; t < TI; t++) ones2_pos[t] = ones2[t];
    };
    const int n_pos_lo = PAIR ? p.n_pos_lo : p.n_pos;

    // src: this lane's column of the staged row (word w at src[w * 32]); xs: the row operands' words of that row
    // (entry t at xs[t * RG_ROWSTRIDE + w])
    constexpr int RG_ROWSTRIDE = Ring<W>::RPC * W;
    auto do_row = [&](const int r, const u64* __restrict__ src, const u64* __restrict__ xs) {
        u64 a[W], m[W];
        const size_t kb = (size_t)r * W;
#pragma unroll
        for (int w = 0; w < W; w++) a[w] = src[w * 32];
        // NH keys of this row's words (warp-uniform constant loads): word k uses KEY[k mod 64] and KEY[k mod 64 + 1]
        u64 key0[W], key1[W];
        if (NH) {
#pragma unroll
            for (int w = 0; w < W; w++) {
                // when hash blocks end on stage boundaries no row straddles a block: one base + constant offsets
                const u32 pk = Ring<W>::CHUNK_FOLD ? (((u32)kb & 63u) + w) : (((u32)kb + w) & 63u);
                key0[w] = c_nh.k[pk];
                key1[w] = c_nh.k[pk + 1];
            }
        }
#pragma unroll
        for (int w = 0; w < W; w++) m[w] = NEEDM ? ld_nc(p.masks + kb + w) : 0ull;
#pragma unroll
        for (int t = 0; t < TI; t++) {
            u64 b[W], out[W];
#pragma unroll
            for (int w = 0; w < W; w++) b[w] = BIN ? xs[t * RG_ROWSTRIDE + w] : 0ull;
            if (!BIN) apply_slot<OP, W, PAIR>(t, out, a, a, m);
            else if (XL) apply_slot<OP, W, PAIR>(t, out, a, b, m);
            else apply_slot<OP, W, PAIR>(t, out, b, a, m);
            if (REWRITE) {
                if (pd[t]) {
#pragma unroll
                    for (int w = 0; w < W; w++) pd[t][(kb + w) * 32] = out[w];
                }
                continue;
            }
            asm("mad.hi.u32 %0, %1, 2, %0;" : "+r"(ones[t]) : "r"((u32)(out[0] >> 32)));
            if (PAIR) asm("mad.hi.u32 %0, %1, 2, %0;" : "+r"(ones2[t]) : "r"((u32)out[0]));
            if (NH) {
#pragma unroll
                for (int w = 0; w < W; w++) {  // oracle fp_nh
                    const u32 xl = (u32)out[w], xh = (u32)(out[w] >> 32);
                    h0[t] = mad_wide(xl + (u32)key0[w], xh + (u32)(key0[w] >> 32), h0[t]);
                    h1[t] = mad_wide(xl + (u32)key1[w], xh + (u32)(key1[w] >> 32), h1[t]);
                    if (!Ring<W>::CHUNK_FOLD) {
                        const u64 k1 = kb + w + 1;
                        if ((k1 & 63) == 0 || k1 == (u64)n) {
                            const u64 u = (((k1 - 1) >> 6) + p.blk_base + 1) * K_STEP;
                            s0[t] += mix64(h0[t] ^ u);
                            s1[t] += mix64(h1[t] + u);
                            h0[t] = h1[t] = 0;
                        }
                    }
                }
            } else if (MUELLER) {
#pragma unroll
                for (int w = 0; w < W; w++) {  // reference _speedups.pyx:196-202
                    u64 mm = mix64_hot(out[w] ^ (tw + (u64)w * K_STEP));
                    h0[t] = (h0[t] ^ mm) * K_FOLD0;
                    h1[t] = (h1[t] ^ ((mm << 32) | (mm >> 32))) * K_FOLD1;
                    if (!Ring<W>::CHUNK_FOLD) {  // per-word block boundary check (rows straddle hash blocks)
                        const u64 k1 = kb + w + 1;
                        if ((k1 & 63) == 0 || k1 == (u64)n) {
                            if (((k1 - 1) >> 6) + p.blk_base == 0) {
                                s0[t] += h0[t];
                                s1[t] += h1[t];
                            } else {
                                s0[t] += mix64(h0[t]);
                                s1[t] += mix64(h1[t]);
                            }
                            h0[t] = K_SEED0;
                            h1[t] = K_SEED1;
                        }
                    }
                }
            } else {
                int dd = d;
                while (dd < p.n_dep && p.deps[dd].k < kb + W) {
                    const Deposit dp = p.deps[dd];
                    u64 word = out[0];
#pragma unroll
                    for (int w = 1; w < W; w++)
                        if (dp.k - kb == (size_t)w) word = out[w];
                    const u64 v = (word >> dp.rsh) & dp.mask;
                    if (dp.pos >= 64) s0[t] += v << (dp.pos - 64);
                    else {
                        s1[t] += v << dp.pos;
                        if (dp.pos > 0) s0[t] += v >> (64 - dp.pos);
                    }
                    dd++;
                }
                if (t == TI - 1) d = dd;
            }
        }
        if (MUELLER) tw += (u64)W * K_STEP;
    };

    // ---- stream the lane operand through the shared-memory ring
    typedef Ring<W> RG;
    const int rows_total = r1 - r0;
    const int nchunks = (rows_total + RG::RPC - 1) / RG::RPC;
    const u64* __restrict__ gsrc = p.cms + ((size_t)lg * (size_t)n + (size_t)r0 * W) * 32;
    // one stage = the lane operand's next RPC rows (one bulk copy issued by lane 0) + the same rows of the
    // TI row operands (strided in memory: one 8-byte cp.async per lane); all 32 lanes take part
    const int my_t = lane / RG_ROWSTRIDE, my_i = lane - my_t * RG_ROWSTRIDE;
    const u64* __restrict__ my_row = (BIN && my_t < TI) ? p.cms + cm_index(row0 + my_t, n, 0) : nullptr;
    auto issue = [&](const int c, const int s) {
        const int rows_c = min(RG::RPC, rows_total - c * RG::RPC);
        u64* stage_base = sbuf + s * RG::STAGE_U64;
        if (lane == 0) {
            const u32 bytes = (u32)rows_c * W * 256u;
            mbar_expect_tx(bars + s, bytes);
            bulk_g2s(stage_base, gsrc + (size_t)c * RG::LANE_U64, bytes, bars + s);
        }
        if (BIN) {
            if (my_row && my_i < rows_c * W)
                cp_async8(stage_base + RG::LANE_U64 + lane, my_row + ((size_t)(r0 + c * RG::RPC) * W + my_i) * 32);
            cp_async_arrive(bars + s);
        }
    };
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < RG::STAGES; s++) mbar_init(bars + s, BIN ? 33 : 1);
        fence_mbar_init();
        fence_async_smem();
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < RG::STAGES; s++)
        if (s < nchunks) issue(s, s);
    int stage = 0;
    u32 parity = 0;
    for (int c = 0; c < nchunks; c++) {
        mbar_wait(bars + stage, parity);
        const u64* __restrict__ src = sbuf + stage * RG::STAGE_U64 + lane;
        const u64* __restrict__ xsrc = sbuf + stage * RG::STAGE_U64 + RG::LANE_U64;
        const int rbase = r0 + c * RG::RPC;
        const int rows_c = min(RG::RPC, r1 - rbase);
        const bool straddle = (p.n_pos > rbase && p.n_pos < rbase + rows_c) ||
                              (PAIR && n_pos_lo > rbase && n_pos_lo < rbase + rows_c);
        if (rbase == p.n_pos) snapshot();
        if (PAIR && rbase == n_pos_lo) snapshot_lo();
        if (rows_c == RG::RPC && !straddle) {
            // partial unroll: a fully unrolled stage of a 4-slot tile is ~24 KB of code, and a level with many
            // small pieces runs a dozen tile variants per SM -- ncu showed `no_instructions` as the top stall
#pragma unroll kRowUnroll
            for (int rr = 0; rr < RG::RPC; rr++) do_row(rbase + rr, src + rr * W * 32, xsrc + rr * W);
        } else {
            for (int rr = 0; rr < rows_c; rr++) {
                if (rr && rbase + rr == p.n_pos) snapshot();
                if (PAIR && rr && rbase + rr == n_pos_lo) snapshot_lo();
                do_row(rbase + rr, src + rr * W * 32, xsrc + rr * W);
            }
        }
        if (HASHED && RG::CHUNK_FOLD) {
            const int rend = rbase + rows_c;
            if ((((u32)rend * W) & 63u) == 0 || rend == p.R) fold(((u32)rend * W - 1) >> 6);
        }
        __syncwarp();
        if (c + RG::STAGES < nchunks) {
            if (lane == 0) fence_async_smem();
            issue(c + RG::STAGES, stage);
        }
        if (++stage == RG::STAGES) {
            stage = 0;
            parity ^= 1u;
        }
    }

    // ---- per-candidate epilogue
    if (REWRITE) return;
    u32 err[TI];
    {
        const int npos_here = max(0, min(r1, p.n_pos) - r0);  // positive rows of this split
#pragma unroll
        for (int t = 0; t < TI; t++) {
            if (p.n_pos >= r1) ones_pos[t] = ones[t];  // every row of the split is positive
            err[t] = ((u32)npos_here - ones_pos[t]) + (ones[t] - ones_pos[t]);
            if (PAIR) {
                const int npos_lo_here = max(0, min(r1, n_pos_lo) - r0);
                if (n_pos_lo >= r1) ones2_pos[t] = ones2[t];
                err[t] += ((u32)npos_lo_here - ones2_pos[t]) + (ones2[t] - ones2_pos[t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < TI; t++) {
        u64 c;
        if (!slot_rank(t, &c)) continue;
        if (p.nsplit > 1) {
            atomicAdd(p.acc + 3 * c, s0[t]);
            atomicAdd(p.acc + 3 * c + 1, s1[t]);
            if (err[t]) atomicAdd(p.acc + 3 * c + 2, (u64)err[t]);
        } else if (p.defer) {  // row shard, no row split: this warp is the only writer of the candidate's sums
            p.acc[3 * c] = s0[t];
            p.acc[3 * c + 1] = s1[t];
            p.acc[3 * c + 2] = (u64)err[t];
        } else {
            finish_candidate<HASHED>(p, c, s0[t], s1[t], err[t]);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// phase A kernel

// Resident CTAs per SM asked of ptxas.  One-word rows keep every hot loop spill-free below 85 registers (checked in
// the SASS), and with 16 warps per SM ncu showed `wait` (fixed-latency dependencies) as the top stall, so W = 1 runs
// 3 CTAs = 24 warps per SM (bench: k_screen 16.4 -> 14.8 ms per search; 4 CTAs: 15.5 ms; re-measured after the NOT pass
// moved into phase B: 2 / 3 / 4 CTAs = 9.65 / 9.86 / 10.50 ms on the bench, 77.3 / 75.8 ms on the 8192-row deep run); wider rows hold whole
// rows in registers and stay at 2.
#ifndef LTL_MIN_CTAS_W1
#define LTL_MIN_CTAS_W1 3
#endif
#ifndef LTL_MIN_CTAS_REWRITE
#define LTL_MIN_CTAS_REWRITE 3  // (4 CTAs -- 64 registers, 4 x 55.5 KB of rings per SM -- measured: 10.3 -> 10.9 ms on config 4)
#endif
template <int W, int KIND, bool PAIR = false>
__global__ void __launch_bounds__(LTL_CTA, (W == 1 ? (KIND == KIND_REWRITE ? LTL_MIN_CTAS_REWRITE : LTL_MIN_CTAS_W1) : 2))
    k_screen(const __grid_constant__ ScreenParams p) {
    static_assert(!PAIR || (W == 1 && (KIND == KIND_NH || KIND == KIND_REWRITE)), "half-width rows: one word, NH fingerprint");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    u64* sbuf = reinterpret_cast<u64*>(smem_raw) + warp * Ring<W>::WARP_U64;
    u64* bars = reinterpret_cast<u64*>(smem_raw) + LTL_WARPS_PER_CTA * Ring<W>::WARP_U64 + warp * Ring<W>::STAGES;
    // Warps are numbered over (tile, row split), split fastest, so that every CTA is full even when a level has few
    // tiles AND the warps of a CTA (and of the CTAs resident beside it) run the same tile variant on different row
    // ranges: with the splits of one tile far apart, the six warps of an SM sub-partition ran six different variants of
    // ~4 KB each through a ~6 KB L0 instruction cache, and ncu showed `no_instruction` as the top stall of every
    // row-split launch (46 % of the samples on BASELINE config 4, cost level 5).
    const i64 gw = (i64)blockIdx.x * LTL_WARPS_PER_CTA + warp;
    int split = 0;
    i64 T = p.tile_offset + gw;
    if (p.nsplit > 1 && KIND != KIND_REWRITE) {
        const i64 tl = gw / p.nsplit;
        split = (int)(gw - tl * p.nsplit);
        T = p.tile_offset + tl;
    } else if (p.nsplit > 1) {
        // the tile-shaped phase B keeps (row split, tile): neighbouring tiles write neighbouring winners, whose partial
        // lines meet in L2 only if they are written at about the same time (tile-major: 10.0 -> 14.5 ms on config 4)
        const i64 launch_tiles = p.total_tiles - p.tile_offset;
        split = (int)(gw / launch_tiles);
        T = p.tile_offset + (gw - (i64)split * launch_tiles);
        if (split >= p.nsplit) return;
    }
    if (T >= p.total_tiles) return;
    // piece of this tile: last piece with tile_base <= T
    int lo = 0, hi = p.n_pieces - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (p.pieces[mid].tile_base <= T) lo = mid;
        else hi = mid - 1;
    }
    const Piece pc = p.pieces[lo];
    const i64 t = T - pc.tile_base;
    i64 rt, lgi;
    {
        // tile order inside a piece keeps ranks monotone: (row tile, lane group) row-major, but for a swapped
        // RECT (lanes over the left operand i, which is the major rank index) lane-group-major
        const bool lane_major = pc.kind == PIECE_RECT && pc.swap;
        const i64 minor = lane_major ? pc.tiles_row : pc.tiles_lane;
        i64 hi_, lo_;
        if ((u64)t < 0xFFFFFFFFull && (u64)minor < 0xFFFFFFFFull) {
            hi_ = (u32)t / (u32)minor;
            lo_ = (u32)t - (u32)hi_ * (u32)minor;
        } else {
            hi_ = t / minor;
            lo_ = t - hi_ * minor;
        }
        rt = lane_major ? lo_ : hi_;
        lgi = lane_major ? hi_ : lo_;
    }
    const i64 lg = pc.lane_g0 + lgi;
    i64 row0 = 0;
    int nv = 1;
    if (pc.kind != PIECE_UNARY) {
        const i64 org = (pc.kind == PIECE_RECT && pc.swap) ? pc.j0 : pc.i0;
        const i64 end = (pc.kind == PIECE_RECT && pc.swap) ? pc.j1 : pc.i1;
        row0 = org + rt * pc.ti;
        nv = (int)min((i64)pc.ti, end - row0);
        if (pc.kind == PIECE_TRI && lg * 32 + 31 <= row0) return;  // tile entirely on/below the diagonal
    }
    // a solver with a lower rank than anything in this tile makes the tile irrelevant
    u64 sol = ~0ull, fuse_off = 0;
    if (p.check_solve && p.mode == MODE_INSERT) {
        i64 ci, cj;
        const i64 lfirst = lg * 32;
        if (pc.kind == PIECE_UNARY) {
            ci = max(lfirst, pc.i0);
            cj = -1;
        } else if (pc.kind == PIECE_RECT && pc.swap) {
            ci = max(lfirst, pc.i0);
            cj = row0;
        } else if (pc.kind == PIECE_RECT) {
            ci = row0;
            cj = max(lfirst, pc.j0);
        } else {
            ci = row0;
            cj = max(lfirst, row0 + 1);
        }
        const u64 cmin = piece_rank(pc, ci, cj);
        sol = *((volatile u64*)&p.ctl->solver_c);
        if (sol < cmin) {
            // the tile's slots stay unwritten: the resolve pass never looks above the solver
            return;
        }
        fuse_off = (u64)(ci - pc.i0);
    }
    const bool xl = pc.swap != 0;

#define LTL_TILE(OP_, TI_, XL_) tile_eval<W, KIND, OP_, TI_, XL_, PAIR>(p, pc, row0, lg, split, lane, sbuf, bars)
#define LTL_TILE_TI(OP_, XL_)                       \
    do {                                            \
        if (W == 1 && KIND != KIND_BITS) {          \
            switch (nv) {                           \
                case 1: LTL_TILE(OP_, 1, XL_); break; \
                case 2: LTL_TILE(OP_, 2, XL_); break; \
                case 3: LTL_TILE(OP_, 3, XL_); break; \
                default: LTL_TILE(OP_, 4, XL_); break; \
            }                                       \
        } else {                                    \
            LTL_TILE(OP_, 1, XL_);                  \
        }                                           \
    } while (0)

    if (W == 1 && KIND != KIND_BITS && pc.kind == PIECE_UNARY && pc.nfuse > 1) {
        // connectives whose every candidate of this tile ranks above a known solver are dropped (they form a
        // suffix: fused connectives are consecutive in enumeration order)
        int nf = pc.nfuse;
        while (nf > 1 && (u64)pc.fcbase[nf - 1] + fuse_off > sol) nf--;
        const int fops = pc.fops & ((1 << (4 * nf)) - 1);
        switch (fops) {
            case OP_NOT: LTL_TILE(OP_NOT, 1, false); break;
            case OP_NEXT: LTL_TILE(OP_NEXT, 1, false); break;
            case OP_FINALLY: LTL_TILE(OP_FINALLY, 1, false); break;
            case OP_GLOBALLY: LTL_TILE(OP_GLOBALLY, 1, false); break;
            case 0x41: LTL_TILE(0x41, 2, false); break;
            case 0x51: LTL_TILE(0x51, 2, false); break;
            case 0x61: LTL_TILE(0x61, 2, false); break;
            case 0x54: LTL_TILE(0x54, 2, false); break;
            case 0x64: LTL_TILE(0x64, 2, false); break;
            case 0x65: LTL_TILE(0x65, 2, false); break;
            case 0x541: LTL_TILE(0x541, 3, false); break;
            case 0x641: LTL_TILE(0x641, 3, false); break;
            case 0x651: LTL_TILE(0x651, 3, false); break;
            case 0x654: LTL_TILE(0x654, 3, false); break;
            case 0x6541: LTL_TILE(0x6541, 4, false); break;
            default: break;
        }
        return;
    }
    switch (pc.op) {
        case OP_IDENT: LTL_TILE(OP_IDENT, 1, false); break;
        case OP_NOT: LTL_TILE(OP_NOT, 1, false); break;
        case OP_NEXT: LTL_TILE(OP_NEXT, 1, false); break;
        case OP_FINALLY: LTL_TILE(OP_FINALLY, 1, false); break;
        case OP_GLOBALLY: LTL_TILE(OP_GLOBALLY, 1, false); break;
        case OP_AND: LTL_TILE_TI(OP_AND, false); break;
        case OP_OR: LTL_TILE_TI(OP_OR, false); break;
        case OP_UNTIL:
            if (xl) LTL_TILE_TI(OP_UNTIL, true);
            else LTL_TILE_TI(OP_UNTIL, false);
            break;
        default: break;
    }
#undef LTL_TILE_TI
#undef LTL_TILE
}

// ------------------------------------------------------------------------------------------------
// phase A for small passes (one-word rows)
//
// k_screen is ~54 K instructions of specialised tiles; a pass of a few hundred candidates touches a long path through it
// once, and ncu shows `no_instruction` (instruction-cache misses) as its top stall by far: 25 us per launch whatever the
// work (config 1: every cost level; every config: its first five or six levels).  This kernel does the same arithmetic
// with a few hundred instructions: one thread per (candidate, block of 64 rows), operands read straight from the entry
// store (consecutive candidates share their left operand and read consecutive right operands), connective chosen by a
// switch, partial sums combined with atomics like any row-split pass.  Bit-identical results: same connectives
// (semantics.cuh), same fingerprint definitions as tile_eval, same finish_candidate.
// one row of a one-word connective chosen at run time
template <int OP_DUMMY = 0>
__device__ __forceinline__ u64 small_apply(const int op, const u64 x, const u64 y, const u64 m) {
    u64 xs[1] = {x}, ys[1] = {y}, ms[1] = {m}, out[1];
    switch (op) {
        case OP_NOT: apply_row<OP_NOT, 1>(out, xs, ys, ms); break;
        case OP_AND: apply_row<OP_AND, 1>(out, xs, ys, ms); break;
        case OP_OR: apply_row<OP_OR, 1>(out, xs, ys, ms); break;
        case OP_NEXT: apply_row<OP_NEXT, 1>(out, xs, ys, ms); break;
        case OP_FINALLY: apply_row<OP_FINALLY, 1>(out, xs, ys, ms); break;
        case OP_GLOBALLY: apply_row<OP_GLOBALLY, 1>(out, xs, ys, ms); break;
        case OP_UNTIL: apply_row<OP_UNTIL, 1>(out, xs, ys, ms); break;
        default: out[0] = x; break;
    }
    return out[0];
}

// rows [r0, r1) of ONE candidate op(x [, y]) over one-word rows: classification errors of those rows and their share of
// the two fingerprint sums (hash blocks are 64 rows: r0 is a multiple of 64 and r1 - r0 <= 64 or the range is whole
// blocks).  NC: the operands are read through the non-coherent path (they were written by an earlier launch); the
// device-resident level loop (levels.cuh) reads matrices written by the running kernel and passes false.
// U rows are loaded before the first of them is used: a thread walks its rows alone, so the loop is bound by the
// latency of its loads (L2: every small pass reads matrices the previous launch / phase wrote), not by their number
template <int KIND, bool NC, int U>
__device__ __forceinline__ void small_rows(const ScreenParams& p, const int op, const u64* __restrict__ px, const u64* __restrict__ py,
                                           const int r0, const int r1, u64& s0, u64& s1, u32& err) {
    constexpr bool NH = KIND == KIND_NH, MUELLER = KIND == KIND_MUELLER, HASHED = NH || MUELLER;
    u64 h0 = NH ? 0ull : K_SEED0, h1 = NH ? 0ull : K_SEED1;
    int d = 0;
    if (KIND == KIND_BITS) {
        int a = 0, b = p.n_dep;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (p.deps[mid].k < (u32)r0) a = mid + 1;
            else b = mid;
        }
        d = a;
    }
    const bool binary = py != px;
    for (int rb = r0; rb < r1; rb += U) {
        u64 xv[U], yv[U], mv[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int r = min(rb + k, r1 - 1);
            xv[k] = NC ? ld_nc(px + (size_t)r * 32) : __ldcg(px + (size_t)r * 32);
            yv[k] = !binary ? 0ull : NC ? ld_nc(py + (size_t)r * 32) : __ldcg(py + (size_t)r * 32);
            mv[k] = ld_nc(p.masks + r);
        }
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int r = rb + k;
            if (r >= r1) break;
            const u64 v = small_apply(op, xv[k], binary ? yv[k] : xv[k], mv[k]);
            const u32 bit = (u32)(v >> 63);
            err += r < p.n_pos ? 1u - bit : bit;  // reference _speedups.pyx:327-333
            if (NH) {  // oracle fp_nh
                const u32 pk = (u32)r & 63u;
                const u64 key0 = c_nh.k[pk], key1 = c_nh.k[pk + 1];
                const u32 xl = (u32)v, xh = (u32)(v >> 32);
                h0 = mad_wide(xl + (u32)key0, xh + (u32)(key0 >> 32), h0);
                h1 = mad_wide(xl + (u32)key1, xh + (u32)(key1 >> 32), h1);
            } else if (MUELLER) {  // reference _speedups.pyx:196-202, blocked
                const u64 mm = mix64(v ^ (((u64)p.blk_base * 64ull + (u64)r + 1ull) * K_STEP));
                h0 = (h0 ^ mm) * K_FOLD0;
                h1 = (h1 ^ ((mm << 32) | (mm >> 32))) * K_FOLD1;
            } else {  // gather / fkp deposits (reference _speedups.pyx:188-195, 205-222)
                while (d < p.n_dep && p.deps[d].k <= (u32)r) {
                    const Deposit dp = p.deps[d];
                    const u64 w = (v >> dp.rsh) & dp.mask;
                    if (dp.pos >= 64) s0 += w << (dp.pos - 64);
                    else {
                        s1 += w << dp.pos;
                        if (dp.pos > 0) s0 += w >> (64 - dp.pos);
                    }
                    d++;
                }
            }
            if (HASHED && ((((u32)r + 1u) & 63u) == 0 || r + 1 == p.R)) {  // the hash block ends with this word
                const u32 blk = ((u32)r >> 6) + p.blk_base;
                if (NH) {
                    const u64 u = (u64)(blk + 1) * K_STEP;
                    s0 += mix64(h0 ^ u);
                    s1 += mix64(h1 + u);
                    h0 = h1 = 0;
                } else {
                    s0 += blk == 0 ? h0 : mix64(h0);
                    s1 += blk == 0 ? h1 : mix64(h1);
                    h0 = K_SEED0;
                    h1 = K_SEED1;
                }
            }
        }
    }
}

// NH over ONE hash block (rows [r0, r1), r0 a multiple of 64, r1 <= r0 + 64) by a group of 8 neighbouring lanes: lane `sub`
// takes rows r0 + sub, r0 + sub + 8, ...  The block's two NH accumulators are sums of products and the error count is a
// sum, so the lanes' partial sums are combined with three shuffle steps; every lane of the group returns the block's
// contribution (s0, s1, err) -- bit-identical to small_rows<KIND_NH>.  All 32 lanes of the warp must call it (`valid` false:
// no loads).  A thread that walks 64 rows alone is bound by the latency of its dependent instructions (~1.5 us per 4 rows
// measured in the level loop); eight rows per lane leave 1/8 of that chain.
template <bool NC>
__device__ __forceinline__ void small_block_nh8(const ScreenParams& p, const int op, const u64* __restrict__ px,
                                                const u64* __restrict__ py, const int r0, const int r1, const int sub,
                                                const bool valid, u64& s0, u64& s1, u32& err) {
    const bool binary = py != px;
    u64 h0 = 0, h1 = 0;
    u32 e = 0;
#pragma unroll
    for (int half = 0; half < 2; half++) {
        u64 xv[4], yv[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int r = r0 + sub + 8 * (4 * half + k);
            const bool in = valid && r < r1;
            xv[k] = !in ? 0ull : NC ? ld_nc(px + (size_t)r * 32) : __ldcg(px + (size_t)r * 32);
            yv[k] = !(in && binary) ? 0ull : NC ? ld_nc(py + (size_t)r * 32) : __ldcg(py + (size_t)r * 32);
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int r = r0 + sub + 8 * (4 * half + k);
            if (!(valid && r < r1)) continue;
            const u64 v = small_apply(op, xv[k], binary ? yv[k] : xv[k], ld_nc(p.masks + r));
            const u32 bit = (u32)(v >> 63);
            e += r < p.n_pos ? 1u - bit : bit;  // reference _speedups.pyx:327-333
            const u32 pk = (u32)r & 63u;  // oracle fp_nh
            const u64 key0 = c_nh.k[pk], key1 = c_nh.k[pk + 1];
            const u32 xl = (u32)v, xh = (u32)(v >> 32);
            h0 = mad_wide(xl + (u32)key0, xh + (u32)(key0 >> 32), h0);
            h1 = mad_wide(xl + (u32)key1, xh + (u32)(key1 >> 32), h1);
        }
    }
#pragma unroll
    for (int d = 4; d >= 1; d >>= 1) {
        h0 += __shfl_xor_sync(0xFFFFFFFFu, h0, d);
        h1 += __shfl_xor_sync(0xFFFFFFFFu, h1, d);
        e += __shfl_xor_sync(0xFFFFFFFFu, e, d);
    }
    const u64 u = (u64)(((u32)r0 >> 6) + p.blk_base + 1) * K_STEP;
    s0 = mix64(h0 ^ u);
    s1 = mix64(h1 + u);
    err = e;
}

// k_screen_small for the NH fingerprint: 8 lanes per (candidate, block of 64 rows)
template <int KIND>  // (KIND_NH only; a template so that every translation unit may see the definition)
__global__ void __launch_bounds__(256) k_screen_small_nh8(const __grid_constant__ ScreenParams p, const u64 total) {
    static_assert(KIND == KIND_NH, "the 8-lane split needs a fingerprint that is a sum over rows");
    const int sub = threadIdx.x & 7;
    const u64 c = (u64)blockIdx.x * 32 + (threadIdx.x >> 3);
    bool valid = c < total;
    int op = 0;
    i64 i = 0, j = -1;
    if (valid) {
        int lo = 0, hi = p.n_pieces - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((u64)p.pieces[mid].cbase <= c) lo = mid;
            else hi = mid - 1;
        }
        const Piece& pc = p.pieces[lo];
        if (pc.ext) valid = false;  // evaluated by phase B of the entries it ranges over (fused NOT)
        else {
            piece_unrank(pc, c, &i, &j);
            op = pc.op;
        }
    }
    const i64 n = p.n;
    const int r0 = (int)blockIdx.y * LTL_SPLIT_ROWS, r1 = min(p.R, r0 + LTL_SPLIT_ROWS);
    const u64* __restrict__ px = p.cms + cm_index(i, n, 0);
    const u64* __restrict__ py = j >= 0 ? p.cms + cm_index(j, n, 0) : px;
    u64 s0, s1;
    u32 err;
    small_block_nh8<true>(p, op, px, py, r0, r1, sub, valid, s0, s1, err);
    if (!valid || sub != 0) return;
    if (p.nsplit > 1 || p.defer) {
        atomicAdd(p.acc + 3 * c, s0);
        atomicAdd(p.acc + 3 * c + 1, s1);
        if (err) atomicAdd(p.acc + 3 * c + 2, (u64)err);
    } else {
        finish_candidate<true>(p, c, s0, s1, err);
    }
}

template <int KIND>
__global__ void __launch_bounds__(256) k_screen_small(const __grid_constant__ ScreenParams p, const u64 total) {
    constexpr bool HASHED = KIND == KIND_NH || KIND == KIND_MUELLER;
    const u64 c = (u64)blockIdx.x * 256 + threadIdx.x;
    if (c >= total) return;
    int lo = 0, hi = p.n_pieces - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((u64)p.pieces[mid].cbase <= c) lo = mid;
        else hi = mid - 1;
    }
    const Piece& pc = p.pieces[lo];
    if (pc.ext) return;  // evaluated by phase B of the entries it ranges over (fused NOT)
    i64 i, j;
    piece_unrank(pc, c, &i, &j);
    const i64 n = p.n;
    const int r0 = (int)blockIdx.y * p.rows_per_split, r1 = min(p.R, r0 + p.rows_per_split);
    const u64* __restrict__ px = p.cms + cm_index(i, n, 0);
    const u64* __restrict__ py = j >= 0 ? p.cms + cm_index(j, n, 0) : px;
    u64 s0 = 0, s1 = 0;
    u32 err = 0;
    small_rows<KIND, true, 8>(p, pc.op, px, py, r0, r1, s0, s1, err);
    if (p.nsplit > 1 || p.defer) {
        atomicAdd(p.acc + 3 * c, s0);
        atomicAdd(p.acc + 3 * c + 1, s1);
        if (err) atomicAdd(p.acc + 3 * c + 2, (u64)err);
    } else {
        finish_candidate<HASHED>(p, c, s0, s1, err);
    }
}

// Small passes over rows of W = 2, 4, 8 or 16 words (NH fingerprint): one lane per (candidate, row).  The row is the unit
// of the connectives (carries run through its W words), the 64-word hash block the unit of the fingerprint: a block is
// 64 / W whole rows, i.e. 64 / W neighbouring lanes, which combine their sums with shuffles; the blocks' sums meet in the
// partial-sum array like the row splits of any pass.  (The tile kernel spent 0.1-0.2 ms on each of the first five cost
// levels of BASELINE config 3 -- a dozen to a few thousand candidates -- whatever the work.)
template <int W>
__global__ void __launch_bounds__(256) k_screen_small_rows(const __grid_constant__ ScreenParams p, const u64 total) {
    static_assert(W > 1 && W <= 16 && 64 % W == 0, "rows must tile the 64-word hash blocks");
    constexpr int LPB = 64 / W;  // lanes (rows) per hash block
    const int l = threadIdx.x & 63;
    const u64 c = (u64)blockIdx.x * 4 + (threadIdx.x >> 6);
    bool valid = c < total;
    int op = 0;
    i64 i = 0, j = -1;
    if (valid) {
        int lo = 0, hi = p.n_pieces - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((u64)p.pieces[mid].cbase <= c) lo = mid;
            else hi = mid - 1;
        }
        const Piece& pc = p.pieces[lo];
        if (pc.ext) valid = false;
        else {
            piece_unrank(pc, c, &i, &j);
            op = pc.op;
        }
    }
    const int r = (int)blockIdx.y * LTL_SPLIT_ROWS + l;
    const bool in = valid && r < p.R;
    const size_t kb = (size_t)r * W;
    u64 h0 = 0, h1 = 0;
    u32 e = 0;
    if (in) {
        const i64 n = p.n;
        const u64* __restrict__ px = p.cms + cm_index(i, n, 0);
        const u64* __restrict__ py = j >= 0 ? p.cms + cm_index(j, n, 0) : px;
        u64 x[W], y[W], m[W], out[W];
#pragma unroll
        for (int w = 0; w < W; w++) {
            x[w] = ld_nc(px + (kb + w) * 32);
            y[w] = j >= 0 ? ld_nc(py + (kb + w) * 32) : 0ull;
            m[w] = ld_nc(p.masks + kb + w);
        }
        switch (op) {
            case OP_NOT: apply_row<OP_NOT, W>(out, x, y, m); break;
            case OP_AND: apply_row<OP_AND, W>(out, x, y, m); break;
            case OP_OR: apply_row<OP_OR, W>(out, x, y, m); break;
            case OP_NEXT: apply_row<OP_NEXT, W>(out, x, y, m); break;
            case OP_FINALLY: apply_row<OP_FINALLY, W>(out, x, y, m); break;
            case OP_GLOBALLY: apply_row<OP_GLOBALLY, W>(out, x, y, m); break;
            case OP_UNTIL: apply_row<OP_UNTIL, W>(out, x, y, m); break;
            default: apply_row<OP_IDENT, W>(out, x, y, m); break;
        }
        const u32 bit = (u32)(out[0] >> 63);
        e = r < p.n_pos ? 1u - bit : bit;  // reference _speedups.pyx:327-333
        const u32 pk0 = (u32)kb & 63u;     // the row lies inside one hash block: no wrap of the key index
#pragma unroll
        for (int w = 0; w < W; w++) {  // oracle fp_nh
            const u64 key0 = c_nh.k[pk0 + w], key1 = c_nh.k[pk0 + w + 1];
            const u32 xl = (u32)out[w], xh = (u32)(out[w] >> 32);
            h0 = mad_wide(xl + (u32)key0, xh + (u32)(key0 >> 32), h0);
            h1 = mad_wide(xl + (u32)key1, xh + (u32)(key1 >> 32), h1);
        }
    }
#pragma unroll
    for (int d = LPB / 2; d >= 1; d >>= 1) {
        h0 += __shfl_xor_sync(0xFFFFFFFFu, h0, d);
        h1 += __shfl_xor_sync(0xFFFFFFFFu, h1, d);
        e += __shfl_xor_sync(0xFFFFFFFFu, e, d);
    }
    if (!in || (l & (LPB - 1))) return;  // the block's first row speaks for it (rows ascend: it is valid if any is)
    const u64 u = (u64)((u32)(kb >> 6) + p.blk_base + 1) * K_STEP;
    atomicAdd(p.acc + 3 * c, mix64(h0 ^ u));
    atomicAdd(p.acc + 3 * c + 1, mix64(h1 + u));
    if (e) atomicAdd(p.acc + 3 * c + 2, (u64)e);
}

// Phase B of a small pass over multi-word rows: one lane per (new entry, row), from the entry's record.  (The tile-shaped
// phase B has the tile kernel's ~50 us minimum; BASELINE config 3 paid it on each of its first four cost levels.)
template <int W>
__global__ void __launch_bounds__(256) k_materialize_small_rows(const __grid_constant__ MaterializeParams p) {
    const i64 k = (i64)blockIdx.x * 4 + (threadIdx.x >> 6);
    const int r = (int)blockIdx.y * LTL_SPLIT_ROWS + (threadIdx.x & 63);
    if (k >= p.count || r >= p.R) return;
    const i64 dst = p.n_base + k;
    const int op = (int)p.rec_op[dst];
    const i64 lhs = p.rec_lhs[dst], rhs = p.rec_rhs[dst];
    const i64 n = p.n;
    const size_t kb = (size_t)r * W;
    const u64* __restrict__ px = p.cms + cm_index(lhs, n, 0);
    const u64* __restrict__ py = p.cms + cm_index(rhs >= 0 ? rhs : lhs, n, 0);
    u64* __restrict__ po = p.cms + cm_index(dst, n, 0);
    u64 x[W], y[W], m[W], out[W];
#pragma unroll
    for (int w = 0; w < W; w++) {
        x[w] = ld_nc(px + (kb + w) * 32);
        y[w] = rhs >= 0 ? ld_nc(py + (kb + w) * 32) : 0ull;
        m[w] = ld_nc(p.masks + kb + w);
    }
    switch (op) {
        case OP_NOT: apply_row<OP_NOT, W>(out, x, y, m); break;
        case OP_AND: apply_row<OP_AND, W>(out, x, y, m); break;
        case OP_OR: apply_row<OP_OR, W>(out, x, y, m); break;
        case OP_NEXT: apply_row<OP_NEXT, W>(out, x, y, m); break;
        case OP_FINALLY: apply_row<OP_FINALLY, W>(out, x, y, m); break;
        case OP_GLOBALLY: apply_row<OP_GLOBALLY, W>(out, x, y, m); break;
        case OP_UNTIL: apply_row<OP_UNTIL, W>(out, x, y, m); break;
        default: apply_row<OP_IDENT, W>(out, x, y, m); break;
    }
#pragma unroll
    for (int w = 0; w < W; w++) po[(kb + w) * 32] = out[w];
}

// ------------------------------------------------------------------------------------------------
// phase B kernel

template <int W, int OP, bool PAIR>
__device__ __forceinline__ void mat_rows(const MaterializeParams& p, const bool mine, const i64 dst, const int lhs,
                                         const int rhs, const int r0, const int r1) {
    constexpr bool BIN = !(OP == OP_IDENT || OP == OP_NOT || OP == OP_NEXT || OP == OP_FINALLY || OP == OP_GLOBALLY);
    constexpr bool NEEDM = (OP == OP_NOT || OP == OP_GLOBALLY);
    if (!mine) return;
    const i64 n = p.n;
    const u64* __restrict__ px = p.cms + cm_index(lhs, n, 0);
    const u64* __restrict__ py = p.cms + cm_index(BIN ? rhs : lhs, n, 0);
    u64* __restrict__ po = p.cms + cm_index(dst, n, 0);
#pragma unroll 4
    for (int r = r0; r < r1; r++) {
        const size_t kb = (size_t)r * W;
        u64 x[W], y[W], m[W], out[W];
#pragma unroll
        for (int w = 0; w < W; w++) {
            x[w] = ld_nc(px + (kb + w) * 32);
            y[w] = BIN ? ld_nc(py + (kb + w) * 32) : 0ull;
            m[w] = NEEDM ? ld_nc(p.masks + kb + w) : 0ull;
        }
        apply_row<OP, W, PAIR>(out, x, y, m);
#pragma unroll
        for (int w = 0; w < W; w++) __stcs(po + (kb + w) * 32, out[w]);  // streaming: next read is a cost level away
    }
}

// group handled by warp `widx` of a phase-B launch (MaterializeParams: processing order), or -1 past the end
__device__ __forceinline__ i64 mat_group(const MaterializeParams& p, const i64 widx) {
    if (p.n_seg == 0) return (p.n_base >> 5) + widx;
    if (widx >= (i64)p.seg_goff[p.n_seg]) return -1;
    int lo = 0, hi = p.n_seg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((i64)p.seg_goff[mid] <= widx) lo = mid;
        else hi = mid - 1;
    }
    return (p.n_base >> 5) + (i64)p.seg_g0[lo] + (widx - (i64)p.seg_goff[lo]);
}

template <int W, bool PAIR = false>
__global__ void __launch_bounds__(LTL_CTA) k_materialize(const __grid_constant__ MaterializeParams p) {
    const int lane = threadIdx.x & 31;
    const i64 g = mat_group(p, (i64)blockIdx.x * LTL_WARPS_PER_CTA + (threadIdx.x >> 5));
    const i64 dst = g * 32 + lane;
    if (g < 0 || g * 32 >= p.n_base + p.count) return;
    const bool valid = dst >= p.n_base && dst < p.n_base + p.count;
    const int op = valid ? (int)p.rec_op[dst] : -1;
    const int lhs = valid ? p.rec_lhs[dst] : 0;
    const int rhs = valid ? p.rec_rhs[dst] : 0;
    const int r0 = blockIdx.y * p.rows_per_split;
    const int r1 = min(p.R, r0 + p.rows_per_split);
    unsigned remaining = __ballot_sync(0xFFFFFFFFu, valid);
    while (remaining) {
        const int leader = __ffs(remaining) - 1;
        const int cur = __shfl_sync(0xFFFFFFFFu, op, leader);
        const bool mine = valid && op == cur;
        remaining &= ~__ballot_sync(0xFFFFFFFFu, mine);
        switch (cur) {
            case OP_NOT: mat_rows<W, OP_NOT, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_AND: mat_rows<W, OP_AND, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_OR: mat_rows<W, OP_OR, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_NEXT: mat_rows<W, OP_NEXT, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_FINALLY: mat_rows<W, OP_FINALLY, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_GLOBALLY: mat_rows<W, OP_GLOBALLY, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            case OP_UNTIL: mat_rows<W, OP_UNTIL, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
            default: mat_rows<W, OP_IDENT, PAIR>(p, mine, dst, lhs, rhs, r0, r1); break;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------------
// phase B with the next level's NOT fused in (one-word rows)
//
// Phase B is bound by HBM (it writes every new matrix once) and leaves the integer pipes idle, while the first
// thing the next cost level does with the new entries is a pass that reads them all back to screen NOT(entry)
// (connective order formula.py:24).  Here that candidate is evaluated from the row that is in registers anyway:
// error count (reference _speedups.pyx:327-333), fingerprint fold (KIND_MUELLER: _speedups.pyx:196-202, blocked;
// KIND_NH: oracle fp_nh), and at the end the same table filing as phase A.  Rows go in blocks of 64 (the
// fingerprint's block length) so the block epilogue stays out of the row loop.

#ifndef LTL_MATF_UNROLL
#define LTL_MATF_UNROLL 16
#endif
#ifndef LTL_MATF_MINB
#define LTL_MATF_MINB 2
#endif
// the evaluate-only twin (closed store gate): nothing is written, so the launch is bound by issue and latency, not by HBM
// writes -- more resident warps, shorter unroll
#ifndef LTL_MATF_EVAL_UNROLL
#define LTL_MATF_EVAL_UNROLL 8
#endif
#ifndef LTL_MATF_EVAL_MINB
#define LTL_MATF_EVAL_MINB 3
#endif

template <int FK>
struct NotFold {
    u64 s0, s1, h0, h1;
    u32 err;
    __device__ __forceinline__ void begin_block() {
        h0 = FK == KIND_NH ? 0ull : K_SEED0;
        h1 = FK == KIND_NH ? 0ull : K_SEED1;
    }
    // v = word k (= row k, W = 1) of NOT(entry); pk = k mod 64
    // (half-width store: v holds two rows; positive_lo says whether the low-half row is a positive trace)
    template <bool PAIR>
    __device__ __forceinline__ void word(const u64 v, const u32 k, const u32 pk, const bool positive, const bool positive_lo) {
        const u32 bit = (u32)(v >> 63);
        err += positive ? 1u - bit : bit;
        if (PAIR) {
            const u32 bit2 = ((u32)v) >> 31;
            err += positive_lo ? 1u - bit2 : bit2;
        }
        if (FK == KIND_NH) {
            const u64 key0 = c_nh.k[pk], key1 = c_nh.k[pk + 1];
            const u32 xl = (u32)v, xh = (u32)(v >> 32);
            h0 = mad_wide(xl + (u32)key0, xh + (u32)(key0 >> 32), h0);
            h1 = mad_wide(xl + (u32)key1, xh + (u32)(key1 >> 32), h1);
        } else {
            const u64 mm = mix64(v ^ ((u64)(k + 1) * K_STEP));  // k: global word index
            h0 = (h0 ^ mm) * K_FOLD0;
            h1 = (h1 ^ ((mm << 32) | (mm >> 32))) * K_FOLD1;
        }
    }
    __device__ __forceinline__ void end_block(const u32 blk) {
        if (FK == KIND_NH) {
            const u64 u = (u64)(blk + 1) * K_STEP;
            s0 += mix64(h0 ^ u);
            s1 += mix64(h1 + u);
        } else {
            s0 += blk == 0 ? h0 : mix64(h0);
            s1 += blk == 0 ? h1 : mix64(h1);
        }
    }
};

template <int OP, int FK, bool PAIR, bool STORE>
__device__ __forceinline__ void mat_rows_not(const MaterializeParams& p, const bool mine, const i64 dst,
                                             const int lhs, const int rhs, NotFold<FK>& f) {
    constexpr bool BIN = !(OP == OP_IDENT || OP == OP_NOT || OP == OP_NEXT || OP == OP_FINALLY || OP == OP_GLOBALLY);
    if (!mine) return;
    const i64 n = p.n;
    const u64* __restrict__ px = p.cms + cm_index(lhs, n, 0);
    const u64* __restrict__ py = p.cms + cm_index(BIN ? rhs : lhs, n, 0);
    u64* __restrict__ po = p.cms + cm_index(dst, n, 0);
    const u64* __restrict__ pm = p.masks;
    const int R = p.R, n_pos = p.n_pos, n_pos_lo = p.n_pos_lo;
    const u32 kbase = p.blk_base * 64u;
    auto row = [&](const int r, const u32 pk) {
        u64 x[1], y[1], m[1], out[1];
        x[0] = ld_nc(px + (size_t)r * 32);
        y[0] = BIN ? ld_nc(py + (size_t)r * 32) : 0ull;
        m[0] = ld_nc(pm + r);
        apply_row<OP, 1, PAIR>(out, x, y, m);
        if (STORE) __stcs(po + (size_t)r * 32, out[0]);  // streaming store: keeps the operand blocks in L2
        f.template word<PAIR>(~out[0] & m[0], kbase + (u32)r, pk, r < n_pos, r < n_pos_lo);
    };
    constexpr int UNROLL = STORE ? LTL_MATF_UNROLL : LTL_MATF_EVAL_UNROLL;
    for (int rb = 0; rb < R; rb += 64) {
        f.begin_block();
        if (rb + 64 <= R) {
#pragma unroll UNROLL
            for (int i = 0; i < 64; i++) row(rb + i, (u32)i);
        } else {
            for (int i = 0; rb + i < R; i++) row(rb + i, (u32)i);
        }
        f.end_block(((u32)rb >> 6) + p.blk_base);
    }
}

// STORE = false: the evaluate-only twin.  A gated pass launches both; each returns at once unless the gate is its way.
template <int FK, bool PAIR = false, bool STORE = true>
__global__ void __launch_bounds__(LTL_CTA, STORE ? LTL_MATF_MINB : LTL_MATF_EVAL_MINB)
    k_materialize_not(const __grid_constant__ MaterializeParams p, const __grid_constant__ ScreenParams sp) {
    // (the gate is a snapshot taken before this launch: candidates filed here may lower ctl->solver_c, never the gate)
    if (p.store_gate != nullptr && (ld_nc(p.store_gate) == ~0ull) != STORE) return;
    const int lane = threadIdx.x & 31;
    const i64 g = mat_group(p, (i64)blockIdx.x * LTL_WARPS_PER_CTA + (threadIdx.x >> 5));
    const i64 dst = g * 32 + lane;
    if (g < 0 || g * 32 >= p.n_base + p.count) return;
    const bool valid = dst >= p.n_base && dst < p.n_base + p.count;
    const int op = valid ? (int)p.rec_op[dst] : -1;
    const int lhs = valid ? p.rec_lhs[dst] : 0;
    const int rhs = valid ? p.rec_rhs[dst] : 0;
    NotFold<FK> f;
    f.s0 = f.s1 = 0;
    f.err = 0;
    unsigned remaining = __ballot_sync(0xFFFFFFFFu, valid);
    while (remaining) {
        const int leader = __ffs(remaining) - 1;
        const int cur = __shfl_sync(0xFFFFFFFFu, op, leader);
        const bool mine = valid && op == cur;
        remaining &= ~__ballot_sync(0xFFFFFFFFu, mine);
        switch (cur) {
            case OP_NOT: mat_rows_not<OP_NOT, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_AND: mat_rows_not<OP_AND, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_OR: mat_rows_not<OP_OR, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_NEXT: mat_rows_not<OP_NEXT, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_FINALLY: mat_rows_not<OP_FINALLY, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_GLOBALLY: mat_rows_not<OP_GLOBALLY, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            case OP_UNTIL: mat_rows_not<OP_UNTIL, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
            default: mat_rows_not<OP_IDENT, FK, PAIR, STORE>(p, mine, dst, lhs, rhs, f); break;
        }
        __syncwarp();
    }
    if (valid) {  // file NOT(dst) as candidate not_cbase + (dst - not_i0) of the pass in flight
        const u64 c = (u64)p.not_cbase + (u64)(dst - p.not_i0);
        if (sp.nsplit > 1) {  // the pass combines row splits: hand the sums to k_finalize
            atomicAdd(sp.acc + 3 * c, f.s0);
            atomicAdd(sp.acc + 3 * c + 1, f.s1);
            if (f.err) atomicAdd(sp.acc + 3 * c + 2, (u64)f.err);
        } else if (sp.defer) {  // row shard: this lane folded all local rows of the entry
            sp.acc[3 * c] = f.s0;
            sp.acc[3 * c + 1] = f.s1;
            sp.acc[3 * c + 2] = (u64)f.err;
        } else {
            finish_candidate<true>(sp, c, f.s0, f.s1, f.err);
        }
    }
}

#endif  // __CUDACC__

// launchers, one translation unit per W (screen_inst.cu compiled with -DLTL_W=<W>)
// (W == 1 has a second pair of launchers for the half-width store: ltl_launch_screen_w1p / ltl_launch_materialize_w1p)
typedef void (*screen_launch_fn)(const ScreenParams&, int kind, dim3 grid, cudaStream_t stream);
typedef void (*materialize_launch_fn)(const MaterializeParams&, const ScreenParams&, int fuse_kind, dim3 grid, cudaStream_t stream);
