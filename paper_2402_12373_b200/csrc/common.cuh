// common.cuh -- shared device/host definitions for the B200 screening core (sm_100a only).
//
// Data layout in HBM:
//   * characteristic matrices ("entries") are stored in GROUPS of 32 entries, word-major inside a
//     group:  word k (k = row*W + w, 0 <= k < n = R*W) of entry e lives at
//         cms[((e >> 5) * n + k) * 32 + (e & 31)]
//     so the 32 lanes of a warp that own the 32 entries of a group read/write one aligned 256-byte
//     line per word (fully coalesced, 8 sectors).
//   * the uniqueness set is an open-addressing table of 32-byte slots {lo, hi, rank, pad}: one
//     DRAM sector per probe.  key = 126-bit fingerprint (top 2 bits of hi always 0, reference
//     kernels.py:35), EMPTY key = all ones.  rank = global enumeration rank of the candidate that
//     owns the key (atomicMin => "lowest enumeration rank wins" = the sequential reference's
//     first-wins admission, _speedups.pyx:245-262), ~0 = key present but not a member.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;
typedef long long i64;

// opcodes (reference formula.py:13-20); 0 doubles as "identity" for add_entry / fingerprint_of.
enum { OP_IDENT = 0, OP_NOT = 1, OP_AND = 2, OP_OR = 3, OP_NEXT = 4, OP_FINALLY = 5, OP_GLOBALLY = 6, OP_UNTIL = 7 };
enum { VAR_GATHER = 0, VAR_MUELLER = 1, VAR_FKP = 2, VAR_NH = 3, VAR_NH32 = 4 };  // NH / NH32: this build's hashes beyond the reference's domain
enum { PIECE_UNARY = 0, PIECE_RECT = 1, PIECE_TRI = 2 };
enum { MODE_INSERT = 0, MODE_FP_ONLY = 1, MODE_LOOKUP = 2, MODE_REWRITE = 3 };
enum { KIND_BITS = 0, KIND_MUELLER = 1, KIND_REWRITE = 2, KIND_NH = 3 };  // what a k_screen instantiation does with a row

#define LTL_GROUP 32
#define LTL_NONE 0xFFFFFFFFu
#define LTL_RANK_NONE 0xFFFFFFFFFFFFFFFFull
#define LTL_WARPS_PER_CTA 8
#define LTL_CTA (32 * LTL_WARPS_PER_CTA)
#define LTL_MAX_W 16
#define LTL_SPLIT_ROWS 64  // row-split granularity: 64 rows = a whole number of 64-word hash blocks

// fingerprint constants (reference kernels.py:28-35)
#define K_MIX1 0xBF58476D1CE4E5B9ull
#define K_MIX2 0x94D049BB133111EBull
#define K_STEP 0x9E3779B97F4A7C15ull
#define K_FOLD0 0xC2B2AE3D27D4EB4Full
#define K_FOLD1 0x9E3779B185EBCA87ull
#define K_SEED0 0x243F6A8885A308D3ull
#define K_SEED1 0x13198A2E03707344ull
#define K_HI_CLEAR 0x3FFFFFFFFFFFFFFFull

struct __align__(32) Slot {
    u64 lo, hi;  // key (16-byte aligned: one ATOMG.CAS.128)
    u64 rank;    // owner's global enumeration rank
    u64 pad;
};

// One run of candidates inside a chunk, in enumeration order (host: plan_chunk in core.cu).
//   UNARY: candidates op(i),      i in [i0, i1)                 rank = cbase + (i - i0)
//   RECT : candidates op(i, j),   i in [i0, i1), j in [j0, j1)  rank = cbase + (i - i0)*(j1 - j0) + (j - j0)
//   TRI  : candidates op(i, j),   i in [i0, i1), j in (i, j1)   rank = cbase + T(i - i0) + (j - i - 1),
//          T(q) = q*m - q*(q-1)/2 with m = j1 - 1 - i0  (reference _speedups.pyx:364-368: i ascending, then j)
// Warp tiles: 32 lanes run over one 32-entry storage group of the "lane operand" (j, or i for
// UNARY / swapped RECT), and up to `ti` consecutive entries of the other operand are applied per lane.
struct Piece {
    int op;
    int kind;       // PIECE_*
    int swap;       // RECT only: lanes run over the left operand i, row tiles over j
    int ti;         // max rows per warp tile (1..4)
    int seg;        // index of the caller's segment this piece belongs to
    int owns_tiles; // 0: a fused sibling, evaluated by the primary unary piece of its range -- or (ext) by phase B
    int ext;        // UNARY NOT over entries whose matrices are written in this very pass: k_materialize evaluates it
    int pad_;
    i64 i0, i1;
    i64 j0, j1;
    i64 cbase;      // chunk-local rank of this piece's first candidate
    i64 count;      // candidates in this piece
    i64 tile_base;  // first warp tile of this piece in the launch
    i64 tiles_lane; // lane groups spanned
    i64 tiles_row;  // row tiles (ceil(rows / ti)); tile t = (row tile, lane group), ordered so that the lowest
                    // rank of a tile never decreases with t: row-major, except swapped RECT (lane-group-major)
    i64 lane_g0;    // first lane group (entry index >> 5)
    // fused unary tiles: the unary connectives of one level all read the same operand bucket, so the first
    // unary piece of a range evaluates up to 4 of them per pass (its siblings then own no tiles).
    int nfuse;      // 0/1: plain piece; >= 2: number of fused connectives
    int fops;       // their opcodes, one nibble each, in enumeration order
    i64 fcbase[4];  // chunk-local rank base of each fused connective's piece
};

// One deposit of the "bits" fingerprints (gather / fkp): take ((word[k] >> rsh) & mask) and add it
// into the 128-bit fingerprint at bit position pos (reference _speedups.pyx:188-195, 205-222).
// Deposits target disjoint bit ranges, so integer addition == bitwise or.
struct Deposit {
    u32 k;
    u32 rsh;
    u64 mask;
    u32 pos;
    u32 pad;
};

// Device-resident control block of one chunk.
struct Ctl {
    u64 solver_c;      // min chunk-local rank whose error count <= err_max (atomicMin), ~0 if none
    u64 oom_c;         // chunk-local rank of the first new unique that does not fit the budget, ~0 if none
    u64 total;         // winners below the solver cutoff
    u64 fp_hi, fp_lo;  // MODE_FP_ONLY / MODE_LOOKUP result for single-candidate queries
    u64 found;
    u64 gate;          // solver_c as it stood when the conditional phase B of this pass was issued (MaterializeParams::store_gate)
    u64 pad;
};

struct ScreenParams {
    const u64* cms;  // entry store (group layout)
    const u64* masks;  // n words
    const Piece* pieces;
    int n_pieces;
    int R, W, n_pos, err_max;  // half-width store: R = stored words per entry (row pairs), n_pos = positive HIGH-half rows
    int n_pos_lo;              // half-width store: positive LOW-half rows (floor(n_pos / 2) of the real rows); else unused
    int pair;                  // 1: half-width store (two 32-bit rows per word, see semantics.cuh apply_pair)
    i64 n;  // words per entry
    i64 total_tiles;
    i64 tile_offset;   // first warp tile of this launch (a level's phase A is issued in several launches)
    int nsplit;        // row splits (gridDim.y); > 1 => partial sums go to acc_*, k_finalize completes
    int rows_per_split;  // multiple of LTL_SPLIT_ROWS
    int variant, mask_k, n_dep;
    const Deposit* deps;
    int mode, check_solve;
    Slot* table;
    u64 table_mask;
    u64 gbase;  // global rank of chunk-local rank 0
    u32* slot;  // per candidate: contender slot / NONE
    u64* fp_out;  // MODE_FP_ONLY: 2 words per candidate (hi, lo)
    u64* acc;  // nsplit > 1 or defer: per-candidate partial sums, 3 words each: (s0, s1, errors) -- one contiguous
               // range per range of candidates, so that row shards all-reduce any part of a pass in one call
    Ctl* ctl;
    // KIND_REWRITE (tile-shaped phase B): winners' matrices go to entry n_base + dest[rank]
    const u32* dest;  // per candidate: position among the winners / NONE
    u64* cms_out;     // same buffer as cms
    i64 n_base;
    // row-sharded cores (one GPU holds rows [row_base, row_base + R) of every matrix): this core's first word is word
    // 64 * blk_base of the whole matrix (fingerprint blocks and tweaks are numbered globally), and partial sums always
    // go to acc_* -- they are summed across GPUs before k_finalize completes the candidates
    u32 blk_base;
    int defer;
    // row shards with a sharded uniqueness table: a candidate is filed only by the shard that owns its fingerprint
    // (fp_owner); the winner flags are OR-ed over the shards afterwards.  owner_world <= 1: every key is ours
    int owner_world, owner_rank;
};

struct MaterializeParams {
    u64* cms;  // reads entries < n_base, writes entries [n_base, n_base + count)
    const u64* masks;
    int R, W;
    i64 n;
    i64 n_base, count;
    const unsigned char* rec_op;
    const int* rec_lhs;
    const int* rec_rhs;
    int nsplit, rows_per_split;
    // fused NOT (k_materialize<W, FK != 0>): while a new entry's rows are in registers, the candidate NOT(entry) of
    // the NEXT cost level is evaluated too -- its chunk-local rank is not_cbase + (entry - not_i0)
    int n_pos;
    int n_pos_lo;  // as in ScreenParams (half-width store)
    i64 not_cbase, not_i0;
    u32 blk_base;  // as in ScreenParams
    // Conditional store (fused NOT only): non-null => the matrices are written only if *store_gate == ~0, i.e. if the
    // pass that is being screened had found no solver when this launch was issued.  A search that ends in this pass never
    // reads the newest level's matrices: only NOT(entry), evaluated here from registers, was needed of them.
    const u64* store_gate;
    // Processing order of the 32-entry groups ("phase B order"): n_seg == 0: group k of the launch is group
    // n_base/32 + k; else the launch walks n_seg runs of groups, run s = groups seg_g0[s] .. of length seg_goff[s+1] -
    // seg_goff[s], ordered so that the runs reading the same block of right operands follow one another
    int n_seg;
    const u32* seg_g0;
    const u32* seg_goff;
};

// One family of runs of the phase-B order: the candidates (i, j) of RECT piece `piece` with j inside block jb of the right
// operand bucket (blocks of `block` entries at absolute multiples of it) form run pos_base + jb * stride + off + (i - i0);
// n_jb == 0: the whole piece is one run at pos_base.
struct PlanFam {
    int piece, n_jb;
    i64 n_i;
    i64 block;
    i64 pos_base, stride, off;
    i64 t_base;  // first plan thread of this family (threads enumerate (jb, i) pairs)
};

__host__ __device__ __forceinline__ u64 mix64(u64 x) {  // reference kernels.py:50-57
    x ^= x >> 30;
    x *= K_MIX1;
    x ^= x >> 27;
    x *= K_MIX2;
    x ^= x >> 31;
    return x;
}

// NH fingerprint (VAR_NH): key table KEY[j] = mix64((j+1)*STEP + SEED0), j = 0..64 (definition: oracle/ltl_oracle.c
// fp_nh).  Two Toeplitz-shifted NH accumulators per 64-word block; one 32x32->64 multiply-add each per word.
constexpr u64 mix64_c(u64 x) {
    x ^= x >> 30;
    x *= K_MIX1;
    x ^= x >> 27;
    x *= K_MIX2;
    x ^= x >> 31;
    return x;
}
struct NhKeys {
    u64 k[66];
    constexpr NhKeys() : k{} {
        for (int j = 0; j < 65; j++) k[j] = mix64_c((u64)(j + 1) * K_STEP + K_SEED0);
        k[65] = 0;
    }
};
#ifdef __CUDACC__
static __constant__ NhKeys c_nh = NhKeys();
#endif
static constexpr NhKeys h_nh = NhKeys();

// owner shard of a fingerprint: same integer mix as sharded.py owner_of
__host__ __device__ __forceinline__ int fp_owner(u64 hi, u64 lo, int world) {
    const u64 x = (hi ^ lo) * K_STEP;
    return (int)(((x >> 33) & 0x7FFFFFFFull) % (u64)world);
}

__host__ __device__ __forceinline__ size_t cm_index(i64 e, i64 n, i64 k) {
    return ((size_t)(e >> 5) * (size_t)n + (size_t)k) * LTL_GROUP + (size_t)(e & 31);
}

// T(q) of the TRI rank formula.
__host__ __device__ __forceinline__ u64 tri_before(u64 q, u64 m) { return q * m - ((q * (q - 1)) >> 1); }

#ifdef __CUDACC__
// ---- 128-bit key helpers -----------------------------------------------------------------
struct Key128 {
    u64 lo, hi;
};

__device__ __forceinline__ Key128 ld_key(const Slot* s) {
    Key128 k;
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(k.lo), "=l"(k.hi) : "l"(s) : "memory");
    return k;
}

__device__ __forceinline__ Key128 cas_key(Slot* s, Key128 cmp, Key128 val) {
    Key128 old;
    asm volatile(
        "{\n\t.reg .b128 c, v, o;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.global.cas.b128 o, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, o;\n\t}"
        : "=l"(old.lo), "=l"(old.hi)
        : "l"(cmp.lo), "l"(cmp.hi), "l"(val.lo), "l"(val.hi), "l"(s)
        : "memory");
    return old;
}

__device__ __forceinline__ u64 slot_hash(u64 hi, u64 lo) { return mix64(lo ^ (hi * K_STEP)); }

// Find the slot of key (inserting it if absent).  Keys never change once written, so a stale
// EMPTY read only costs one extra CAS.
__device__ __forceinline__ u64 table_find_or_claim(Slot* table, u64 mask, u64 hi, u64 lo) {
    u64 s = slot_hash(hi, lo) & mask;
    const Key128 empty = {~0ull, ~0ull};
    const Key128 mine = {lo, hi};
    while (true) {
        Key128 k = ld_key(table + s);
        if (k.hi == hi && k.lo == lo) return s;
        if (k.hi == ~0ull) {
            Key128 old = cas_key(table + s, empty, mine);
            if (old.hi == ~0ull || (old.hi == hi && old.lo == lo)) return s;
        }
        s = (s + 1) & mask;
    }
}

// Lookup only: slot index or ~0.
__device__ __forceinline__ u64 table_find(const Slot* table, u64 mask, u64 hi, u64 lo) {
    u64 s = slot_hash(hi, lo) & mask;
    while (true) {
        Key128 k = ld_key(table + s);
        if (k.hi == hi && k.lo == lo) return s;
        if (k.hi == ~0ull) return ~0ull;
        s = (s + 1) & mask;
    }
}

__device__ __forceinline__ u64 ld_rank(const Slot* s) {
    u64 r;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(r) : "l"(&s->rank) : "memory");
    return r;
}

__device__ __forceinline__ u64 ld_nc(const u64* p) { return __ldg(p); }
#endif
