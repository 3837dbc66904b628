// traces.cuh -- device-resident specification ("ltl_traces", include/ltl_core.h): the padded character matrix, the
// row hashes used to screen it for duplicate traces, and after packing the length masks and the propositions'
// characteristic sequences.  Shared between traces.cu (the object) and core.cu (cores created on it).
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

#define LTL_TRACES_INFO 48

struct ltl_traces {
    int device = -1;
    i64 R = 0, n_pos = 0;
    int W = 0, L = 0, Lpad = 0, n_props = 0;  // n_props == 0: not packed yet
    cudaStream_t st = nullptr;
    // one device allocation, carved up: chars (R x Lpad uint16), lengths, masks, atoms, row hashes, scratch
    char* buf = nullptr;       // characters, lengths, row hashes, suspects, counters, hash table
    size_t cap = 0;
    char* pack_buf = nullptr;  // masks + atoms (allocated by ltl_traces_pack)
    size_t pack_cap = 0;
    uint16_t* d_chars = nullptr;
    i64* d_len = nullptr;
    u64* d_masks = nullptr;   // [R * W]
    u64* d_atoms = nullptr;   // [n_props][R * W]
    u64* d_rowhash = nullptr; // [R][2]
    u64* d_info = nullptr;    // LTL_TRACES_INFO words of counters written by the kernels
    i64* d_pairs = nullptr;   // suspects: (row, first row with the same hash)
    i64 pairs_cap = 0;
    Slot* d_table = nullptr;
    u64 table_cap = 0;
    u64 info[LTL_TRACES_INFO] = {0};
    std::vector<i64> suspects;
    u64 h2d_bytes = 0, d2h_bytes = 0;
    std::string err;
};

// info[] layout (ltl_traces_info copies it out)
enum {
    TI_ROWS = 0, TI_NPOS, TI_WORDS, TI_MAXLEN, TI_MINLEN, TI_NONEMPTY, TI_CHAR_OR, TI_POS_POSITIONS, TI_POS_BITS,
    TI_SUSPECTS, TI_EMPTY_POS, TI_NPROPS, TI_H2D, TI_D2H,
    TI_ATOM_ERR = 16,   // [16] misclassified traces of the bare proposition p
    TI_NATOM_ERR = 32,  // [16] ... of its negation
};
