// semantics.cuh -- branch-free LTL connectives on one W-word row of a characteristic matrix.
//
// Position j of a trace lives in word j/64 at bit 63 - j%64 (MSB first), so "the suffix starting one
// step later" is a logical LEFT shift of the whole W-word row; zeros enter from beyond the last word, and
// word 0 is the MOST significant word of the row read as one 64*W-bit integer.
//
// The reference computes F / G / U as O(log n) shift-by-powers-of-two scans with ceil(log2(64*W)) rounds
// (bitsem.py:107-149 for one word, width-generic form bitsem.py:307-334; _speedups.pyx:291-325).  Both are
// closures that move information from later positions to earlier ones, i.e. from LOW bits to HIGH bits --
// the direction an integer adder propagates carries.  The default device formulation therefore lets the
// adder do the scan (results are bit-identical, the parity tests compare against the scan oracle):
//     F x   = x | -x                         all bits at and above the lowest set bit
//     G x   = ~F(~x & m) & m                 (dual inside the length mask, reference bitsem.py:133-138)
//     x U y = y | s | (((x + s) ^ x) & x),   s = x & (y << 1)
//             (a seed s sits where x holds and y holds one step later; adding it to x ripples a carry up
//              through the run of x-ones above it, and the bits the addition flipped are the flooded run)
// which is ~12 instead of ~56 integer instructions per 64-bit word for U (and 4 vs 24 for F); ncu showed
// k_screen ALU-pipe bound at 58 instructions per candidate word with the scans (profiles/README.md).
// Multi-word rows chain the carry from word W-1 up to word 0.  Building with -DLTL_SEMANTICS_SCAN selects
// the reference's scan formulation instead (kept for A/B measurements).
// Everything is fully unrolled over compile-time W: shifts >= 64 become register renames, shifts < 64
// funnel shifts with the neighbouring word.
#pragma once
#include "common.cuh"

template <int W>
struct Rounds {
    static constexpr int value = (64 * W <= 64) ? 6 : (64 * W <= 128) ? 7 : (64 * W <= 256) ? 8 : (64 * W <= 512) ? 9 : 10;
};
static_assert(LTL_MAX_W <= 16, "Rounds<> covers rows of up to 1024 positions");

// word w of (a << S), row-wide
template <int W, int S>
__device__ __forceinline__ u64 shl_word(const u64 (&a)[W], int w) {
    constexpr int q = S >> 6, r = S & 63;
    u64 lo = (w + q < W) ? a[w + q] : 0ull;
    if (r == 0) return lo;
    u64 hi = (w + q + 1 < W) ? a[w + q + 1] : 0ull;
    return (lo << r) | (hi >> ((64 - r) & 63));
}

// c |= c << 2^I for I = 0..ROUNDS-1 (in place; ascending w only reads words >= w, i.e. old values)
template <int W, int I, int ROUNDS>
struct SmearOr {
    static __device__ __forceinline__ void run(u64 (&c)[W]) {
#pragma unroll
        for (int w = 0; w < W; w++) c[w] |= shl_word<W, (1 << I)>(c, w);
        SmearOr<W, I + 1, ROUNDS>::run(c);
    }
};
template <int W, int ROUNDS>
struct SmearOr<W, ROUNDS, ROUNDS> {
    static __device__ __forceinline__ void run(u64 (&)[W]) {}
};

// acc |= run & (acc << s); run &= run << s   (last run update is dead: reference _speedups.pyx:321-324)
template <int W, int I, int ROUNDS>
struct UntilRounds {
    static __device__ __forceinline__ void run(u64 (&acc)[W], u64 (&rn)[W]) {
#pragma unroll
        for (int w = 0; w < W; w++) acc[w] |= rn[w] & shl_word<W, (1 << I)>(acc, w);
        if (I + 1 < ROUNDS) {
#pragma unroll
            for (int w = 0; w < W; w++) rn[w] &= shl_word<W, (1 << I)>(rn, w);
        }
        UntilRounds<W, I + 1, ROUNDS>::run(acc, rn);
    }
};
template <int W, int ROUNDS>
struct UntilRounds<W, ROUNDS, ROUNDS> {
    static __device__ __forceinline__ void run(u64 (&)[W], u64 (&)[W]) {}
};

// out = a + b over the whole row (word W-1 least significant); carries chained upward
template <int W>
__device__ __forceinline__ void row_add(u64 (&out)[W], const u64 (&a)[W], const u64 (&b)[W]) {
    u64 c = 0;
#pragma unroll
    for (int w = W - 1; w >= 0; w--) {
        const u64 t = a[w] + b[w];
        const u64 t2 = t + c;
        c = (u64)(t < a[w]) | (u64)(t2 < t);
        out[w] = t2;
    }
}

// out = x | -x over the whole row: every bit at and above the lowest set bit
template <int W>
__device__ __forceinline__ void row_smear_up(u64 (&out)[W], const u64 (&x)[W]) {
    u64 c = 1;  // -x = ~x + 1
#pragma unroll
    for (int w = W - 1; w >= 0; w--) {
        const u64 t = ~x[w] + c;
        c = c & (u64)(t == 0);
        out[w] = x[w] | t;
    }
}

// ---- half-width rows (PAIR): traces of at most 32 positions are stored TWO ROWS PER 64-BIT WORD -- row 2i in the
// high half, row 2i+1 in the low half (uint32 storage for L <= 32; fingerprint = NH over these words, oracle fp_nh32).
// The connectives act on both halves at once; nothing may cross from the low half into the high one:
//     X   : (x << 1) with bit 32 cleared            F   : x | -x per half (two 32-bit negations)
//     U   : the carry-chain form with two 32-bit adds
__device__ __forceinline__ u64 pack_halves(u32 hi, u32 lo) { return ((u64)hi << 32) | lo; }
#define LTL_PAIR_SHL1_MASK 0xFFFFFFFEFFFFFFFEull

template <int OP>
__device__ __forceinline__ u64 apply_pair(const u64 x, const u64 y, const u64 m) {
    if (OP == OP_IDENT) return x;
    if (OP == OP_NOT) return ~x & m;
    if (OP == OP_AND) return x & y;
    if (OP == OP_OR) return x | y;
    if (OP == OP_NEXT) return (x << 1) & LTL_PAIR_SHL1_MASK;
    if (OP == OP_FINALLY) {
        const u32 h = (u32)(x >> 32), l = (u32)x;
        return pack_halves(h | (0u - h), l | (0u - l));
    }
    if (OP == OP_GLOBALLY) {  // dual of F inside the mask (reference bitsem.py:133-138)
        const u64 t = ~x & m;
        const u32 h = (u32)(t >> 32), l = (u32)t;
        return ~pack_halves(h | (0u - h), l | (0u - l)) & m;
    }
    // OP_UNTIL: y | s | (((x + s) ^ x) & x), s = x & (y << 1), per half
    const u64 sd = x & ((y << 1) & LTL_PAIR_SHL1_MASK);
    const u64 t = pack_halves((u32)(x >> 32) + (u32)(sd >> 32), (u32)x + (u32)sd);
    return y | sd | ((t ^ x) & x);
}

// out = OP(x [, y]) on one row; m = the row's length mask (used by NOT / GLOBALLY only).
// x is the left (or only) operand, y the right operand.  PAIR (W == 1 only): the word holds two 32-bit rows.
template <int OP, int W, bool PAIR = false>
__device__ __forceinline__ void apply_row(u64 (&out)[W], const u64 (&x)[W], const u64 (&y)[W], const u64 (&m)[W]) {
    if (PAIR) {
        out[0] = apply_pair<OP>(x[0], y[0], m[0]);
        return;
    }
    if (OP == OP_IDENT) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = x[w];
    } else if (OP == OP_NOT) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = ~x[w] & m[w];
    } else if (OP == OP_AND) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = x[w] & y[w];
    } else if (OP == OP_OR) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = x[w] | y[w];
    } else if (OP == OP_NEXT) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = shl_word<W, 1>(x, w);
#ifdef LTL_SEMANTICS_SCAN
    } else if (OP == OP_FINALLY) {
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = x[w];
        SmearOr<W, 0, Rounds<W>::value>::run(out);
    } else if (OP == OP_GLOBALLY) {  // dual of F inside the mask (reference bitsem.py:133-138)
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = ~x[w] & m[w];
        SmearOr<W, 0, Rounds<W>::value>::run(out);
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = ~out[w] & m[w];
    } else {  // OP_UNTIL
        u64 rn[W];
#pragma unroll
        for (int w = 0; w < W; w++) {
            out[w] = y[w];
            rn[w] = x[w];
        }
        UntilRounds<W, 0, Rounds<W>::value>::run(out, rn);
    }
#else
    } else if (OP == OP_FINALLY) {
        row_smear_up<W>(out, x);
    } else if (OP == OP_GLOBALLY) {  // dual of F inside the mask (reference bitsem.py:133-138)
        u64 t[W];
#pragma unroll
        for (int w = 0; w < W; w++) t[w] = ~x[w] & m[w];
        row_smear_up<W>(out, t);
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = ~out[w] & m[w];
    } else {  // OP_UNTIL
        u64 sd[W], t[W];
#pragma unroll
        for (int w = 0; w < W; w++) sd[w] = x[w] & shl_word<W, 1>(y, w);
        row_add<W>(t, x, sd);
#pragma unroll
        for (int w = 0; w < W; w++) out[w] = y[w] | sd[w] | ((t[w] ^ x[w]) & x[w]);
    }
#endif
}

__host__ __device__ __forceinline__ bool op_is_unary(int op) {
    return op == OP_IDENT || op == OP_NOT || op == OP_NEXT || op == OP_FINALLY || op == OP_GLOBALLY;
}
__host__ __device__ __forceinline__ bool op_needs_mask(int op) { return op == OP_NOT || op == OP_GLOBALLY; }
