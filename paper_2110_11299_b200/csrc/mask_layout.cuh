// Per-row view of every device mask layout (include/dsa_b200.h dsa_mask):
// ROW_TOPK / COLVEC / BLOCK lists (BLOCK entries expand to `block` keys) and
// the THRESHOLD global CSR.
#pragma once

#include <stdint.h>

#include "kernels.h"

namespace dsa {

struct RowList {
    const uint32_t* cols;
    int count;       // entries in cols
    int expand;      // BLOCK: each entry expands to `expand` keys
};

__device__ __forceinline__ RowList row_list(const AttnArgs& a, int64_t pair, int64_t i) {
    RowList r{nullptr, 0, 1};
    switch (a.mode) {
        case kRowTopk:
            r.cols = a.cols + (pair * a.L + i) * a.keep;
            r.count = static_cast<int>(a.keep);
            break;
        case kColvec: {
            const int64_t nb = (a.L + a.vec_v - 1) / a.vec_v;
            r.cols = a.cols + (pair * nb + i / a.vec_v) * a.keep;
            r.count = static_cast<int>(a.keep);
            break;
        }
        case kBlock: {
            const int64_t nb = (a.L + a.block - 1) / a.block;
            r.cols = a.cols + (pair * nb + i / a.block) * a.keep;
            r.count = static_cast<int>(a.keep);
            r.expand = static_cast<int>(a.block);
            break;
        }
        default: {
            const uint64_t b = a.rowptr[pair * a.L + i], e = a.rowptr[pair * a.L + i + 1];
            r.cols = a.cols + b;
            r.count = static_cast<int>(e - b);
        }
    }
    return r;
}

}  // namespace dsa
