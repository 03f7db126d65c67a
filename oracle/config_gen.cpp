// ORACLE TEST INFRASTRUCTURE -- not part of the product.
//
// The BASELINE config generators (paper_1610_03154_b200/csrc/problems.cpp, pure host
// C++) built into their own CPU library, oracle/build/libconfiggen.so, so that the
// reference arm of bench.py (and any CPU-only caller) can make its inputs without
// loading the GPU library libamgcu.so.  The bytes are the same as amgcu_generate's:
// both call the one generate_config / config_options.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "../paper_1610_03154_b200/csrc/host_common.h"

namespace {
thread_local std::string g_err;

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}
}  // namespace

extern "C" {

const char* gen_last_error(void) { return g_err.c_str(); }
void gen_free(void* p) { std::free(p); }

// same contract as amgcu_generate (include/amgcu.h): malloc'd arrays, freed with gen_free
int gen_generate_config(int32_t config, int32_t n, amgcu_csr* A, int32_t* k, double** B, int32_t* has_left,
                        double** Bhat, double** b) {
    try {
        amgcu::Problem p = amgcu::generate_config(config, n);
        A->n_rows = p.A.n_rows;
        A->n_cols = p.A.n_cols;
        A->nnz = p.A.nnz();
        A->block_size = p.A.block_size;
        A->row_offsets = dup(p.A.row_offsets);
        A->col_indices = dup(p.A.col_indices);
        A->values = dup(p.A.values);
        *k = p.k;
        *B = dup(p.B);
        *has_left = p.has_left ? 1 : 0;
        *Bhat = p.has_left ? dup(p.Bhat) : nullptr;
        *b = dup(p.b);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

int gen_config_options(int32_t config, amgcu_setup_options* so, amgcu_solve_options* vo) {
    try {
        amgcu::config_options(config, so, vo);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // extern "C"
