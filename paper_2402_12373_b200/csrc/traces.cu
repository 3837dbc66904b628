// traces.cu -- the device-resident specification (include/ltl_core.h: ltl_traces_*).
//
// What the reference does on the host before a search, done on the device for specifications of many traces:
//   * duplicate screening of Specification (reference traces.py:64-106: per-side de-duplication, P and N disjoint):
//     every trace is hashed to 128 bits, the hashes are filed in an open-addressing table with atomicMin(row),
//     and rows that are not the first holder of their hash come back as SUSPECTS for an exact comparison on the
//     host (none, normally: then the specification is known to be duplicate-free without a host pass over it);
//   * the census the closed-form overfit cost needs (reference formula.py:230-250) and the widest character;
//   * trace packing (reference bitsem.py:73-88, TraceContext.from_traces; layout rule N2), leaving masks and atoms
//     in HBM for ltl_core_create_on_traces / ltl_core_add_atom -- nothing is copied back;
//   * the atom fast path's error counts (reference enumerator.py:182-192).
#include <algorithm>
#include <cstring>
#include <mutex>

#include "../../include/ltl_core.h"
#include "traces.cuh"

#define LTL_MAX_DEVICES 64

static thread_local std::string g_traces_error;
extern "C" const char* ltl_traces_last_error(const ltl_traces* t) { return t ? t->err.c_str() : g_traces_error.c_str(); }

// ------------------------------------------------------------------------------------------------ kernels

__device__ __forceinline__ u64 rotl64(u64 x, int r) { return (x << r) | (x >> (64 - r)); }

// One thread per (row, word): the 64 characters of the word (128 bytes) -> two chained 64-bit hashes, added into the
// row's pair; characters at positions >= length do not count (equal traces hash equally whatever lies beyond them).
__global__ void __launch_bounds__(256) k_rowhash(const uint16_t* __restrict__ chars, const i64* __restrict__ lengths, i64 R,
                                                 i64 n_pos, int L, int Lpad, int W, u64* __restrict__ rowhash,
                                                 u64* __restrict__ info) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = t < R * W;
    const i64 r = in ? t / W : 0;
    const int w = in ? (int)(t - r * W) : 0;
    const i64 len64 = in ? lengths[r] : 0;
    const int len = len64 < (i64)L ? (int)len64 : L;
    const int live = in ? max(0, min(64, len - w * 64)) : 0;
    u64 a = K_SEED0 ^ ((u64)(w + 1) * K_STEP), b = K_SEED1 + (u64)(w + 1) * K_FOLD1;
    u64 cor = 0;
    u32 bits = 0;
    if (in) {
        const uint4* row = reinterpret_cast<const uint4*>(chars + (size_t)r * Lpad + (size_t)w * 64);
        for (int v = 0; v < 8; v++) {
            if (v * 8 >= live) break;
            const uint4 q4 = __ldg(row + v);
            u64 q[2] = {((u64)q4.y << 32) | q4.x, ((u64)q4.w << 32) | q4.z};
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int nl = max(0, min(4, live - (v * 8 + h * 4)));
                const u64 x = nl >= 4 ? q[h] : (nl > 0 ? q[h] & ((1ull << (16 * nl)) - 1ull) : 0ull);
                a = (a ^ x) * K_FOLD0;
                b = (b ^ rotl64(x, 29)) * K_FOLD1;
                a ^= a >> 29;
                b ^= b >> 31;
                cor |= x;
                bits += __popcll(x);
            }
        }
        u64 hA = mix64(a ^ ((u64)(live + 1) * K_STEP)), hB = mix64(b + (u64)(live + 1) * K_MIX1);
        if (w == 0) {
            hA += mix64((u64)len64 * K_MIX2 + K_SEED1);
            hB += mix64((u64)len64 * K_FOLD0 ^ K_SEED0);
        }
        atomicAdd(rowhash + 2 * r, hA);
        atomicAdd(rowhash + 2 * r + 1, hB);
    }
    // census: widest character, set proposition bits and positions of the positive traces, length range
    u32 c16 = (u32)((cor | (cor >> 16) | (cor >> 32) | (cor >> 48)) & 0xFFFFull);
    const bool pos = in && r < n_pos;
    u32 pbits = pos ? bits : 0u;
    const bool first = in && w == 0;
    u32 plen = (first && pos) ? (u32)len : 0u;
    u32 nonempty = (first && len > 0) ? 1u : 0u, empty_pos = (first && pos && len == 0) ? 1u : 0u;
    u32 mx = first ? (u32)len : 0u, mn = first ? (u32)len : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c16 |= __shfl_xor_sync(0xFFFFFFFFu, c16, o);
        pbits += __shfl_xor_sync(0xFFFFFFFFu, pbits, o);
        plen += __shfl_xor_sync(0xFFFFFFFFu, plen, o);
        nonempty += __shfl_xor_sync(0xFFFFFFFFu, nonempty, o);
        empty_pos += __shfl_xor_sync(0xFFFFFFFFu, empty_pos, o);
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (c16) atomicOr(info + TI_CHAR_OR, (u64)c16);
        if (pbits) atomicAdd(info + TI_POS_BITS, (u64)pbits);
        if (plen) atomicAdd(info + TI_POS_POSITIONS, (u64)plen);
        if (nonempty) atomicAdd(info + TI_NONEMPTY, (u64)nonempty);
        if (empty_pos) atomicAdd(info + TI_EMPTY_POS, (u64)empty_pos);
        atomicMax(info + TI_MAXLEN, (u64)mx);
        if (mn != 0xFFFFFFFFu) atomicMin(info + TI_MINLEN, (u64)mn);
    }
}

// file every row's hash: the lowest row index holding a hash owns it
__global__ void __launch_bounds__(256) k_rowfile(const u64* __restrict__ rowhash, i64 R, Slot* table, u64 mask,
                                                 u32* __restrict__ slot) {
    const i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const u64 hi = rowhash[2 * r] & K_HI_CLEAR, lo = rowhash[2 * r + 1];
    const u64 s = table_find_or_claim(table, mask, hi, lo);
    atomicMin(&table[s].rank, (u64)r);
    slot[r] = (u32)s;
}

// rows that are not the first holder of their hash: (row, first row) pairs for the exact comparison on the host
__global__ void __launch_bounds__(256) k_rowflag(const u32* __restrict__ slot, i64 R, const Slot* __restrict__ table,
                                                 i64* __restrict__ pairs, i64 cap, u64* __restrict__ info) {
    const i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const u64 first = ld_rank(table + slot[r]);
    if (first == (u64)r) return;
    const u64 k = atomicAdd(info + TI_SUSPECTS, 1ull);
    if ((i64)k < cap) {
        pairs[2 * k] = r;
        pairs[2 * k + 1] = (i64)first;
    }
}

// Trace packing from the resident character matrix (reference bitsem.py:73-88; one thread per (row, word), as
// k_pack in core.cu) + the error counts of the bare propositions and their negations (atom fast path).
template <int NP>
__global__ void __launch_bounds__(256) k_pack_dev(const uint16_t* __restrict__ chars, const i64* __restrict__ lengths, i64 R,
                                                 i64 n_pos, int L, int Lpad, int W, int n_props, u64* __restrict__ masks,
                                                 u64* __restrict__ atoms, u64* __restrict__ info) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = t < R * W;
    const i64 r = in ? t / W : 0;
    const int w = in ? (int)(t - r * W) : 0;
    const i64 len64 = in ? lengths[r] : 0;
    const int len = len64 < (i64)L ? (int)len64 : L;
    const int live = in ? max(0, min(64, len - w * 64)) : 0;
    u64 acc[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) acc[p] = 0;
    if (in) {
        const uint16_t* row = chars + (size_t)r * Lpad + (size_t)w * 64;
        for (int v = 0; v < 8 && v * 8 < live; v++) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(row) + v);
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
        masks[t] = live == 0 ? 0ull : (~0ull << ((64 - live) & 63));
        for (int p = 0; p < NP; p++)
            if (p < n_props) atoms[(size_t)p * (size_t)(R * W) + (size_t)t] = acc[p];
    }
    // verdict of the bare proposition / its negation at position 0 (reference bitsem.py:157-160)
    const bool first = in && w == 0;
    const bool pos = r < n_pos;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        if (p >= n_props) break;
        const bool bit = first && (acc[p] >> 63);
        const bool nbit = first && !bit && live > 0;  // (~atom & mask) at position 0
        const unsigned e = __ballot_sync(0xFFFFFFFFu, first && (pos ? !bit : bit));
        const unsigned ne = __ballot_sync(0xFFFFFFFFu, first && (pos ? !nbit : nbit));
        if ((threadIdx.x & 31) == 0) {
            if (e) atomicAdd(info + TI_ATOM_ERR + p, (u64)__popc(e));
            if (ne) atomicAdd(info + TI_NATOM_ERR + p, (u64)__popc(ne));
        }
    }
}

// ------------------------------------------------------------------------------------------------ buffers

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};
static std::mutex g_buf_mutex;
static DevBuf g_cache[LTL_MAX_DEVICES][2];  // [device][0: characters + hashes + table, 1: masks + atoms]

static void* take_buf(int device, int which, size_t need, size_t* cap_out) {
    {
        std::lock_guard<std::mutex> lock(g_buf_mutex);
        DevBuf& c = g_cache[device][which];
        if (c.p && c.cap >= need) {
            void* p = c.p;
            *cap_out = c.cap;
            c = DevBuf();
            return p;
        }
        if (c.p) {
            cudaFree(c.p);
            c = DevBuf();
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, need) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    *cap_out = need;
    return p;
}

static void give_buf(int device, int which, void* p, size_t cap) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lock(g_buf_mutex);
        DevBuf& c = g_cache[device][which];
        if (!c.p) {
            c.p = p;
            c.cap = cap;
            return;
        }
    }
    cudaFree(p);
}

static inline size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }

// ------------------------------------------------------------------------------------------------ C ABI

extern "C" {

void ltl_traces_destroy(ltl_traces* t) {
    if (!t) return;
    if (t->device >= 0) {
        cudaSetDevice(t->device);
        if (t->st) {
            cudaStreamSynchronize(t->st);
            cudaStreamDestroy(t->st);
        }
        give_buf(t->device, 0, t->buf, t->cap);
        give_buf(t->device, 1, t->pack_buf, t->pack_cap);
        cudaGetLastError();
    }
    delete t;
}

int ltl_traces_create(const uint16_t* pos_chars, const int64_t* pos_lengths, int64_t n_pos, const uint16_t* neg_chars,
                      const int64_t* neg_lengths, int64_t n_neg, int L, int device, ltl_traces** out) {
    g_traces_error.clear();
    if (!out) return LTL_ERR_ARG;
    *out = nullptr;
    auto bad = [&](const char* m) {
        g_traces_error = m;
        return LTL_ERR_ARG;
    };
    const i64 R = n_pos + n_neg;
    if (n_pos < 0 || n_neg < 0 || R < 1 || L < 0) return bad("traces: bad shape");
    const int W = std::max(1, (L + 63) / 64);
    if (W > LTL_MAX_W) return bad("traces: rows longer than 1024 positions");
    if ((n_pos && (!pos_chars || !pos_lengths)) || (n_neg && (!neg_chars || !neg_lengths))) return bad("traces: null buffer");
    if (device < 0 || device >= LTL_MAX_DEVICES) return bad("traces: bad device");
    cudaError_t e;
    auto cuda_fail = [&](cudaError_t ce, ltl_traces* t) {
        g_traces_error = std::string("traces: ") + cudaGetErrorString(ce);
        cudaGetLastError();
        ltl_traces_destroy(t);
        return LTL_ERR_CUDA;
    };
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, nullptr);
    ltl_traces* t = new ltl_traces();
    t->device = device;
    t->R = R;
    t->n_pos = n_pos;
    t->W = W;
    t->L = L;
    t->Lpad = 64 * W;
    if ((e = cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, t);
    u64 tcap = 1u << 12;
    while (tcap < (u64)R * 2) tcap <<= 1;
    t->table_cap = tcap;
    t->pairs_cap = std::min<i64>(R, 1 << 20);
    const size_t b_chars = up256((size_t)R * t->Lpad * 2), b_len = up256((size_t)R * 8), b_hash = up256((size_t)R * 16),
                 b_slot = up256((size_t)R * 4), b_pairs = up256((size_t)t->pairs_cap * 16),
                 b_info = up256(LTL_TRACES_INFO * 8), b_table = up256((size_t)tcap * sizeof(Slot));
    const size_t need = b_chars + b_len + b_hash + b_slot + b_pairs + b_info + b_table;
    t->buf = (char*)take_buf(device, 0, need, &t->cap);
    if (!t->buf) {
        g_traces_error = "traces: device memory exhausted";
        ltl_traces_destroy(t);
        return LTL_ERR_DEVICE_OOM;
    }
    char* q = t->buf;
    t->d_chars = (uint16_t*)q;
    q += b_chars;
    t->d_len = (i64*)q;
    q += b_len;
    t->d_rowhash = (u64*)q;
    q += b_hash;
    u32* d_slot = (u32*)q;
    q += b_slot;
    t->d_pairs = (i64*)q;
    q += b_pairs;
    t->d_info = (u64*)q;
    q += b_info;
    t->d_table = (Slot*)q;
    cudaStream_t st = t->st;
    // upload: positives then negatives, rows padded to whole words (the 16-byte loads of the kernels stay in bounds)
    auto upload = [&](const uint16_t* chars, const int64_t* lengths, i64 rows, i64 row0) -> cudaError_t {
        if (!rows) return cudaSuccess;
        cudaError_t ce;
        uint16_t* dst = t->d_chars + (size_t)row0 * t->Lpad;
        if (L == t->Lpad) ce = cudaMemcpyAsync(dst, chars, (size_t)rows * L * 2, cudaMemcpyHostToDevice, st);
        else if (L == 0) ce = cudaSuccess;
        else ce = cudaMemcpy2DAsync(dst, (size_t)t->Lpad * 2, chars, (size_t)L * 2, (size_t)L * 2, (size_t)rows, cudaMemcpyHostToDevice, st);
        if (ce != cudaSuccess) return ce;
        t->h2d_bytes += (size_t)rows * L * 2 + (size_t)rows * 8;
        return cudaMemcpyAsync(t->d_len + row0, lengths, (size_t)rows * 8, cudaMemcpyHostToDevice, st);
    };
    if (L != t->Lpad && (e = cudaMemsetAsync(t->d_chars, 0, (size_t)R * t->Lpad * 2, st)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = upload(pos_chars, pos_lengths, n_pos, 0)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = upload(neg_chars, neg_lengths, n_neg, n_pos)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaMemsetAsync(t->d_rowhash, 0, (size_t)R * 16, st)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaMemsetAsync(t->d_info, 0, LTL_TRACES_INFO * 8, st)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaMemsetAsync(t->d_info + TI_MINLEN, 0xFF, 8, st)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaMemsetAsync(t->d_table, 0xFF, (size_t)tcap * sizeof(Slot), st)) != cudaSuccess) return cuda_fail(e, t);
    const unsigned nbw = (unsigned)(((size_t)R * W + 255) / 256), nbr = (unsigned)((R + 255) / 256);
    k_rowhash<<<nbw, 256, 0, st>>>(t->d_chars, t->d_len, R, n_pos, L, t->Lpad, W, t->d_rowhash, t->d_info);
    k_rowfile<<<nbr, 256, 0, st>>>(t->d_rowhash, R, t->d_table, tcap - 1, d_slot);
    k_rowflag<<<nbr, 256, 0, st>>>(d_slot, R, t->d_table, t->d_pairs, t->pairs_cap, t->d_info);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaMemcpyAsync(t->info, t->d_info, LTL_TRACES_INFO * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, t);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, t);
    t->d2h_bytes += LTL_TRACES_INFO * 8;
    const i64 ns = std::min<i64>((i64)t->info[TI_SUSPECTS], t->pairs_cap);
    if (ns > 0) {
        t->suspects.resize((size_t)ns * 2);
        if ((e = cudaMemcpy(t->suspects.data(), t->d_pairs, (size_t)ns * 16, cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e, t);
        t->d2h_bytes += (size_t)ns * 16;
    }
    t->info[TI_ROWS] = (u64)R;
    t->info[TI_NPOS] = (u64)n_pos;
    t->info[TI_WORDS] = (u64)W;
    *out = t;
    return LTL_OK;
}

int ltl_traces_pack(ltl_traces* t, int n_props) {
    if (!t) return LTL_ERR_ARG;
    if (n_props < 1 || n_props > 16) {
        t->err = "traces: 1..16 propositions";
        return LTL_ERR_ARG;
    }
    cudaError_t e;
    auto cuda_fail = [&](cudaError_t ce) {
        t->err = std::string("traces: ") + cudaGetErrorString(ce);
        cudaGetLastError();
        return LTL_ERR_CUDA;
    };
    if ((e = cudaSetDevice(t->device)) != cudaSuccess) return cuda_fail(e);
    if (t->n_props == n_props) return LTL_OK;
    const size_t words = (size_t)t->R * t->W;
    const size_t need = up256(words * 8) + up256(words * 8 * (size_t)n_props);
    if (t->pack_cap < need) {
        give_buf(t->device, 1, t->pack_buf, t->pack_cap);
        t->pack_buf = (char*)take_buf(t->device, 1, need, &t->pack_cap);
        if (!t->pack_buf) {
            t->pack_cap = 0;
            t->err = "traces: device memory exhausted";
            return LTL_ERR_DEVICE_OOM;
        }
    }
    t->d_masks = (u64*)t->pack_buf;
    t->d_atoms = (u64*)(t->pack_buf + up256(words * 8));
    if ((e = cudaMemsetAsync(t->d_info + TI_ATOM_ERR, 0, 32 * 8, t->st)) != cudaSuccess) return cuda_fail(e);
    const unsigned nb = (unsigned)((words + 255) / 256);
    if (n_props <= 4)
        k_pack_dev<4><<<nb, 256, 0, t->st>>>(t->d_chars, t->d_len, t->R, t->n_pos, t->L, t->Lpad, t->W, n_props, t->d_masks, t->d_atoms, t->d_info);
    else if (n_props <= 8)
        k_pack_dev<8><<<nb, 256, 0, t->st>>>(t->d_chars, t->d_len, t->R, t->n_pos, t->L, t->Lpad, t->W, n_props, t->d_masks, t->d_atoms, t->d_info);
    else
        k_pack_dev<16><<<nb, 256, 0, t->st>>>(t->d_chars, t->d_len, t->R, t->n_pos, t->L, t->Lpad, t->W, n_props, t->d_masks, t->d_atoms, t->d_info);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemcpyAsync(t->info + TI_ATOM_ERR, t->d_info + TI_ATOM_ERR, 32 * 8, cudaMemcpyDeviceToHost, t->st)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamSynchronize(t->st)) != cudaSuccess) return cuda_fail(e);
    t->d2h_bytes += 32 * 8;
    t->n_props = n_props;
    t->info[TI_NPROPS] = (u64)n_props;
    return LTL_OK;
}

int ltl_traces_info(ltl_traces* t, uint64_t out[LTL_TRACES_INFO]) {
    if (!t || !out) return LTL_ERR_ARG;
    t->info[TI_H2D] = t->h2d_bytes;
    t->info[TI_D2H] = t->d2h_bytes;
    memcpy(out, t->info, sizeof(t->info));
    return LTL_OK;
}

int ltl_traces_suspects(ltl_traces* t, int64_t* pairs, int64_t cap_pairs) {
    if (!t || (cap_pairs > 0 && !pairs)) return LTL_ERR_ARG;
    const i64 n = std::min<i64>((i64)t->suspects.size() / 2, cap_pairs);
    if (n > 0) memcpy(pairs, t->suspects.data(), (size_t)n * 16);
    return (int)std::min<i64>(n, 0x7FFFFFFF);
}

int ltl_traces_export(ltl_traces* t, uint64_t* masks_out, uint64_t* atoms_out) {
    if (!t || !masks_out || !atoms_out) return LTL_ERR_ARG;
    if (!t->n_props) {
        t->err = "traces: not packed yet";
        return LTL_ERR_ARG;
    }
    cudaSetDevice(t->device);
    const size_t words = (size_t)t->R * t->W;
    cudaError_t e = cudaMemcpyAsync(masks_out, t->d_masks, words * 8, cudaMemcpyDeviceToHost, t->st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(atoms_out, t->d_atoms, words * 8 * (size_t)t->n_props, cudaMemcpyDeviceToHost, t->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(t->st);
    if (e != cudaSuccess) {
        t->err = std::string("traces: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return LTL_ERR_CUDA;
    }
    t->d2h_bytes += words * 8 * (size_t)(t->n_props + 1);
    return LTL_OK;
}

// ---- trace files (reference traces.py:180-253: one trace per line, positions separated by ';', each position a
// comma-separated 0/1 vector over the alphabet, a '---' line between positives and negatives).  Host code: one pass to
// size the matrices, one to fill them; files that are not in canonical form (any other byte, ragged vectors, stray
// separators) are refused with the line number and left to the caller's line-by-line reader, which owns the messages.
static int trace_file_walk(const char* data, size_t n, int* width_io, int64_t counts[2], int* max_len, int* extra_sections,
                           int64_t* bad_line, uint16_t* chars[2], int64_t* lengths[2], int L) {
    int width = *width_io;
    int section = 0;
    int64_t line_no = 0, rows[2] = {0, 0};
    size_t i = 0;
    int longest = 0;
    while (i < n) {
        line_no++;
        size_t e = i;
        while (e < n && data[e] != '\n') e++;
        size_t a = i, b = e;
        while (b > a && data[b - 1] == '\r') b--;
        i = e + 1;
        if (a == b) continue;  // blank line
        if (data[a] == '-') {
            if (b - a != 3 || data[a + 1] != '-' || data[a + 2] != '-') {
                *bad_line = line_no;
                return LTL_ERR_ARG;
            }
            section++;
            continue;
        }
        // one trace: digits separated by ',' inside a position and ';' between positions
        int positions = 0, in_pos = 0;
        uint16_t ch = 0;
        uint16_t* out = (chars && section < 2) ? chars[section] + (size_t)rows[section] * (size_t)L : nullptr;
        bool expect_digit = true;
        for (size_t k = a; k < b; k++) {
            const char c = data[k];
            if (expect_digit) {
                if (c != '0' && c != '1') {
                    *bad_line = line_no;
                    return LTL_ERR_ARG;
                }
                if (c == '1' && in_pos < 16) ch |= (uint16_t)(1u << in_pos);
                in_pos++;
                expect_digit = false;
            } else {
                if (c == ',') {
                    expect_digit = true;
                } else if (c == ';') {
                    if (width < 0) width = in_pos;
                    if (in_pos != width) {
                        *bad_line = line_no;
                        return LTL_ERR_ARG;
                    }
                    if (out && positions < L) out[positions] = ch;
                    positions++;
                    in_pos = 0;
                    ch = 0;
                    expect_digit = true;
                } else {
                    *bad_line = line_no;
                    return LTL_ERR_ARG;
                }
            }
        }
        if (expect_digit) {  // the line ended in a separator
            *bad_line = line_no;
            return LTL_ERR_ARG;
        }
        if (width < 0) width = in_pos;
        if (in_pos != width || width > 16) {
            *bad_line = line_no;
            return LTL_ERR_ARG;
        }
        if (out && positions < L) out[positions] = ch;
        positions++;
        if (section < 2) {
            if (lengths) lengths[section][rows[section]] = positions;
            rows[section]++;
            longest = std::max(longest, positions);
        }
    }
    *width_io = width;
    counts[0] = rows[0];
    counts[1] = rows[1];
    *max_len = longest;
    *extra_sections = section - 1;
    return LTL_OK;
}

int ltl_trace_file_scan(const char* data, uint64_t n, int64_t counts_out[2], int* max_len, int* width, int* extra_sections,
                        int64_t* bad_line) {
    if ((n && !data) || !counts_out || !max_len || !width || !extra_sections || !bad_line) return LTL_ERR_ARG;
    *bad_line = 0;
    *width = -1;
    return trace_file_walk(data, (size_t)n, width, counts_out, max_len, extra_sections, bad_line, nullptr, nullptr, 0);
}

int ltl_trace_file_fill(const char* data, uint64_t n, int width, int L, uint16_t* pos_chars, int64_t* pos_lengths,
                        uint16_t* neg_chars, int64_t* neg_lengths) {
    if ((n && !data) || width < 1 || L < 0) return LTL_ERR_ARG;
    int64_t counts[2], bad = 0;
    int max_len = 0, extra = 0, w = width;
    uint16_t* chars[2] = {pos_chars, neg_chars};
    int64_t* lengths[2] = {pos_lengths, neg_lengths};
    return trace_file_walk(data, (size_t)n, &w, counts, &max_len, &extra, &bad, chars, lengths, L);
}

}  // extern "C"
