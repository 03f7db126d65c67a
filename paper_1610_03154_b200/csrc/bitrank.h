// Bit-rank helpers of the band-staged masked product's mask-pair records
// (masked_band.cuh), host + device so that tests/cpp/bitrank_check.cpp can check them
// exhaustively against the plain loops.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define BR_HD __host__ __device__ __forceinline__
#else
#define BR_HD inline
#endif

namespace amgcu {
namespace bitrank {

BR_HD int popcount32(unsigned int v) {
#ifdef __CUDA_ARCH__
    return __popc(v);
#else
    return __builtin_popcount(v);
#endif
}

// position of the j-th (0-based) set bit of the 24-bit mask m (j below its popcount)
BR_HD unsigned int nth_set_bit24(unsigned int m, int j) {
    unsigned int pos = 0;
    int c = popcount32(m & 0xfffu);
    if (j >= c) {
        j -= c;
        m >>= 12;
        pos = 12;
    }
    c = popcount32(m & 0x3fu);
    if (j >= c) {
        j -= c;
        m >>= 6;
        pos += 6;
    }
    c = popcount32(m & 0x7u);
    if (j >= c) {
        j -= c;
        m >>= 3;
        pos += 3;
    }
    c = static_cast<int>(m & 1u);
    if (j >= c) {
        j -= c;
        m >>= 1;
        pos += 1;
    }
    c = static_cast<int>(m & 1u);
    if (j >= c) pos += 1;
    return pos;
}

// The match of two sorted column lists as a mask pair: bit s of *mi set when a[s] occurs
// in b, bit q of *mt set when b[q] occurs in a; the j-th set bit of one pairs with the
// j-th of the other (both lists ascending, so the match is monotone).  Returns the count.
BR_HD int match_masks(const int32_t* a, int la, const int32_t* b, int lb, unsigned int* mi, unsigned int* mt) {
    unsigned int x = 0u, y = 0u;
    int q = 0, n = 0;
    for (int s = 0; s < la; ++s) {
        while (q < lb && b[q] < a[s]) ++q;
        if (q < lb && b[q] == a[s]) {
            x |= 1u << s;
            y |= 1u << q;
            ++n;
        }
    }
    *mi = x;
    *mt = y;
    return n;
}

// position in b of a's slot s under the mask pair, or -1
BR_HD int partner(unsigned int mi, unsigned int mt, int s) {
    if (!((mi >> s) & 1u)) return -1;
    return static_cast<int>(nth_set_bit24(mt, popcount32(mi & ((1u << s) - 1u))));
}

}  // namespace bitrank
}  // namespace amgcu
