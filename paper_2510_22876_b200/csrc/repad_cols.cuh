// repad_cols.cuh -- one output column of the out-of-place Alg. 2 Phase 3 repad
// with the §3.1 masks / positions, for K3's gather
// kernel (repad.cu).  (A K1 epilogue that did this itself for B <= 2 was measured slower
// than the separate K3 under PDL -- DESIGN.md negative results.)
#pragma once
#include <cstdint>

namespace specdec {

// E_i[t] for t < emit_i: draft tokens, then the bonus
__device__ __forceinline__ int64_t emitted_token(const int64_t *d, int32_t a, int64_t b, int t) {
    return t < a ? d[t] : b;
}

// Column c (< L' + k) of row i, out of place:
//   c <  p'            : pad (mask 0, position 0)
//   p' <= c < p' + n   : old token at column c - p' + p      (unpad + repad)
//   p' + n <= c < L'   : E[c - p' - n]                        (append A ++ [B])
// A finished row (R9) is a dummy length-1 row: pads, then [pad] at L'-1.
__device__ __forceinline__ void repad_col(int c, int32_t Lnew, int32_t pn, bool fin, int32_t po,
                                          int32_t n, const int64_t *src, int64_t *dst,
                                          int64_t *mrow, int64_t *prow, const int64_t *d,
                                          int32_t a, int64_t b, int64_t pad_id) {
    const bool content = c >= pn;
    mrow[c] = content ? 1 : 0;
    prow[c] = content ? c - pn : 0;
    if (c < Lnew) {
        int64_t t = pad_id;
        if (!fin && content) {
            const int32_t j = c - pn;
            t = j < n ? src[po + j] : emitted_token(d, a, b, j - n);
        }
        dst[c] = t;
    }
}

}  // namespace specdec
