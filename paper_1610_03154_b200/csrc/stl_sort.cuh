// std::sort as GCC's libstdc++ performs it (bits/stl_algo.h, bits/stl_heap.h),
// for use on the device where the reference sorts with an unstable comparator
// and the tie order therefore decides results: ensure_min_support's candidates
// ordered by magnitude (interpolation.hpp:631-632).  Same steps in the same
// order -- introsort with median-of-three partitioning, heapsort once the depth
// limit (2 floor(log2 n)) is spent, final insertion sort with the 16-element
// threshold -- so equal keys end up exactly where the host std::sort puts them.
// `less(a, b)` is the strict weak ordering the reference passes.
#pragma once

#ifndef __CUDACC__  // plain C++ (the host test of the replica)
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#endif

namespace amgcu {
namespace stlsort {

constexpr int kThreshold = 16;

template <typename T>
__host__ __device__ inline void swap_elem(T& a, T& b) {
    T t = a;
    a = b;
    b = t;
}

template <typename T, typename Less>
__host__ __device__ inline void move_median_to_first(T* result, T* a, T* b, T* c, Less less) {
    if (less(*a, *b)) {
        if (less(*b, *c)) swap_elem(*result, *b);
        else if (less(*a, *c)) swap_elem(*result, *c);
        else swap_elem(*result, *a);
    } else if (less(*a, *c)) {
        swap_elem(*result, *a);
    } else if (less(*b, *c)) {
        swap_elem(*result, *c);
    } else {
        swap_elem(*result, *b);
    }
}

template <typename T, typename Less>
__host__ __device__ inline T* unguarded_partition(T* first, T* last, T* pivot, Less less) {
    while (true) {
        while (less(*first, *pivot)) ++first;
        --last;
        while (less(*pivot, *last)) --last;
        if (!(first < last)) return first;
        swap_elem(*first, *last);
        ++first;
    }
}

template <typename T, typename Less>
__host__ __device__ inline void push_heap_(T* first, long hole, long top, T value, Less less) {
    long parent = (hole - 1) / 2;
    while (hole > top && less(first[parent], value)) {
        first[hole] = first[parent];
        hole = parent;
        parent = (hole - 1) / 2;
    }
    first[hole] = value;
}

template <typename T, typename Less>
__host__ __device__ inline void adjust_heap(T* first, long hole, long len, T value, Less less) {
    const long top = hole;
    long second = hole;
    while (second < (len - 1) / 2) {
        second = 2 * (second + 1);
        if (less(first[second], first[second - 1])) --second;
        first[hole] = first[second];
        hole = second;
    }
    if ((len & 1) == 0 && second == (len - 2) / 2) {
        second = 2 * (second + 1);
        first[hole] = first[second - 1];
        hole = second - 1;
    }
    push_heap_(first, hole, top, value, less);
}

template <typename T, typename Less>
__host__ __device__ inline void make_heap_(T* first, T* last, Less less) {
    const long len = last - first;
    if (len < 2) return;
    long parent = (len - 2) / 2;
    while (true) {
        T value = first[parent];
        adjust_heap(first, parent, len, value, less);
        if (parent == 0) return;
        --parent;
    }
}

template <typename T, typename Less>
__host__ __device__ inline void pop_heap_(T* first, T* last, T* result, Less less) {
    T value = *result;
    *result = *first;
    adjust_heap(first, 0L, static_cast<long>(last - first), value, less);
}

// std::__partial_sort(first, last, last): heap select, then sort_heap
template <typename T, typename Less>
__host__ __device__ inline void heap_sort_(T* first, T* last, Less less) {
    make_heap_(first, last, less);
    while (last - first > 1) {
        --last;
        pop_heap_(first, last, last, less);
    }
}

// std::__introsort_loop without recursion (no device stack): libstdc++ recurses into
// [cut, last) and loops on [first, cut); the two ranges are disjoint, so deferring one
// on an explicit stack -- each with the same depth budget -- gives the same result.
template <typename T, typename Less>
__host__ __device__ inline void introsort_loop(T* first, T* last, int depth, Less less) {
    struct Range {
        T* first;
        T* last;
        int depth;
    };
    Range todo[64];
    int top = 0;
    todo[top++] = {first, last, depth};
    while (top > 0) {
        Range r = todo[--top];
        while (r.last - r.first > kThreshold) {
            if (r.depth == 0) {
                heap_sort_(r.first, r.last, less);
                break;
            }
            --r.depth;
            T* mid = r.first + (r.last - r.first) / 2;
            move_median_to_first(r.first, r.first + 1, mid, r.last - 1, less);
            T* cut = unguarded_partition(r.first + 1, r.last, r.first, less);
            todo[top++] = {cut, r.last, r.depth};
            r.last = cut;
        }
    }
}

template <typename T, typename Less>
__host__ __device__ inline void unguarded_linear_insert(T* last, Less less) {
    T val = *last;
    T* next = last - 1;
    while (less(val, *next)) {
        *last = *next;
        last = next;
        --next;
    }
    *last = val;
}

template <typename T, typename Less>
__host__ __device__ inline void insertion_sort(T* first, T* last, Less less) {
    if (first == last) return;
    for (T* i = first + 1; i != last; ++i) {
        if (less(*i, *first)) {
            T val = *i;
            for (T* k = i; k != first; --k) *k = *(k - 1);
            *first = val;
        } else {
            unguarded_linear_insert(i, less);
        }
    }
}

template <typename T, typename Less>
__host__ __device__ inline void sort(T* first, T* last, Less less) {
    if (first == last) return;
    long n = last - first;
    int lg = 0;
    while (n > 1) {
        n >>= 1;
        ++lg;
    }
    introsort_loop(first, last, 2 * lg, less);
    if (last - first > kThreshold) {
        insertion_sort(first, first + kThreshold, less);
        for (T* i = first + kThreshold; i != last; ++i) unguarded_linear_insert(i, less);
    } else {
        insertion_sort(first, last, less);
    }
}

}  // namespace stlsort
}  // namespace amgcu
