// screen_inst.cu -- instantiates the hot kernels for one row width; compiled once per W with -DLTL_W=<W>.
#include "screen.cuh"

#ifndef LTL_W
#error "compile with -DLTL_W=<words per row>"
#endif

#define LTL_CAT2(a, b) a##b
#define LTL_CAT(a, b) LTL_CAT2(a, b)

#ifdef LTL_PAIR
// the half-width store (two 32-bit rows per word; one-word rows, NH fingerprint only): -DLTL_W=1 -DLTL_PAIR
#if LTL_W != 1
#error "LTL_PAIR needs LTL_W == 1"
#endif
extern "C" void ltl_launch_screen_w1p(const ScreenParams& p, int kind, dim3 grid, cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_screen<1, KIND_NH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<1>::CTA_BYTES);
        cudaFuncSetAttribute(k_screen<1, KIND_REWRITE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<1>::CTA_BYTES);
        configured = true;
    }
    if (kind == KIND_NH) k_screen<1, KIND_NH, true><<<grid, LTL_CTA, Ring<1>::CTA_BYTES, stream>>>(p);
    else k_screen<1, KIND_REWRITE, true><<<grid, LTL_CTA, Ring<1>::CTA_BYTES, stream>>>(p);
}
extern "C" void ltl_launch_materialize_w1p(const MaterializeParams& p, const ScreenParams& sp, int fuse_kind, dim3 grid,
                                           cudaStream_t stream) {
    if (fuse_kind == KIND_NH) {
        k_materialize_not<KIND_NH, true><<<grid, LTL_CTA, 0, stream>>>(p, sp);
        if (p.store_gate) k_materialize_not<KIND_NH, true, false><<<grid, LTL_CTA, 0, stream>>>(p, sp);
    } else {
        k_materialize<1, true><<<grid, LTL_CTA, 0, stream>>>(p);
    }
}
#else

extern "C" void LTL_CAT(ltl_launch_screen_w, LTL_W)(const ScreenParams& p, int kind, dim3 grid, cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {  // > 48 KiB of dynamic shared memory needs an opt-in, once per process
        cudaFuncSetAttribute(k_screen<LTL_W, KIND_MUELLER>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<LTL_W>::CTA_BYTES);
        cudaFuncSetAttribute(k_screen<LTL_W, KIND_NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<LTL_W>::CTA_BYTES);
        cudaFuncSetAttribute(k_screen<LTL_W, KIND_BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<LTL_W>::CTA_BYTES);
        cudaFuncSetAttribute(k_screen<LTL_W, KIND_REWRITE>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<LTL_W>::CTA_BYTES);
        configured = true;
    }
    if (kind == KIND_MUELLER) k_screen<LTL_W, KIND_MUELLER><<<grid, LTL_CTA, Ring<LTL_W>::CTA_BYTES, stream>>>(p);
    else if (kind == KIND_NH) k_screen<LTL_W, KIND_NH><<<grid, LTL_CTA, Ring<LTL_W>::CTA_BYTES, stream>>>(p);
    else if (kind == KIND_BITS) k_screen<LTL_W, KIND_BITS><<<grid, LTL_CTA, Ring<LTL_W>::CTA_BYTES, stream>>>(p);
    else k_screen<LTL_W, KIND_REWRITE><<<grid, LTL_CTA, Ring<LTL_W>::CTA_BYTES, stream>>>(p);
}

#if LTL_W == 1
// small passes over one-word rows: the compact kernel (screen.cuh: k_screen_small)
extern "C" void ltl_launch_screen_small(const ScreenParams& p, int kind, unsigned long long total, cudaStream_t stream) {
    dim3 grid((unsigned)((total + 255) / 256), (unsigned)p.nsplit);
    if (kind == KIND_MUELLER) k_screen_small<KIND_MUELLER><<<grid, 256, 0, stream>>>(p, total);
    else if (kind == KIND_NH && p.rows_per_split == LTL_SPLIT_ROWS)  // (always: core.cu cuts small passes into hash blocks)
        k_screen_small_nh8<KIND_NH><<<dim3((unsigned)((total + 31) / 32), (unsigned)p.nsplit), 256, 0, stream>>>(p, total);
    else if (kind == KIND_NH) k_screen_small<KIND_NH><<<grid, 256, 0, stream>>>(p, total);
    else k_screen_small<KIND_BITS><<<grid, 256, 0, stream>>>(p, total);
}
#endif

#if LTL_W == 2 || LTL_W == 4 || LTL_W == 8 || LTL_W == 16
// small NH passes over rows of 2 / 4 / 8 / 16 words (screen.cuh: k_screen_small_rows); sums go to p.acc
extern "C" void LTL_CAT(ltl_launch_screen_small_w, LTL_W)(const ScreenParams& p, unsigned long long total, cudaStream_t stream) {
    k_screen_small_rows<LTL_W><<<dim3((unsigned)((total + 3) / 4), (unsigned)p.nsplit), 256, 0, stream>>>(p, total);
}
#endif

// fuse_kind != 0 (one-word rows only; the host never asks otherwise): phase B that also screens NOT(new entry)
extern "C" void LTL_CAT(ltl_launch_materialize_w, LTL_W)(const MaterializeParams& p, const ScreenParams& sp, int fuse_kind,
                                                          dim3 grid, cudaStream_t stream) {
#if LTL_W == 1
    // (a gated pass launches the storing kernel and its evaluate-only twin: the gate lets exactly one of them run)
    if (fuse_kind == KIND_NH) {
        k_materialize_not<KIND_NH><<<grid, LTL_CTA, 0, stream>>>(p, sp);
        if (p.store_gate) k_materialize_not<KIND_NH, false, false><<<grid, LTL_CTA, 0, stream>>>(p, sp);
        return;
    }
    if (fuse_kind == KIND_MUELLER) {
        k_materialize_not<KIND_MUELLER><<<grid, LTL_CTA, 0, stream>>>(p, sp);
        if (p.store_gate) k_materialize_not<KIND_MUELLER, false, false><<<grid, LTL_CTA, 0, stream>>>(p, sp);
        return;
    }
#endif
    (void)sp;
    (void)fuse_kind;
    k_materialize<LTL_W><<<grid, LTL_CTA, 0, stream>>>(p);
}
#endif  // LTL_PAIR
