// Host-side types shared by the C ABI, the setup/solve orchestration and the
// problem generators of libamgcu.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amgcu.h"

namespace amgcu {

// Exceptions mirror the reference's; the C ABI maps them to
// amgcu_status codes.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct HostCsr {
    int32_t n_rows = 0, n_cols = 0, block_size = 1;
    std::vector<int32_t> row_offsets{0}, col_indices;
    std::vector<double> values;
    int32_t nnz() const { return static_cast<int32_t>(col_indices.size()); }
};

struct Problem {
    HostCsr A;
    int32_t k = 1;
    std::vector<double> B;  // n x k column-major
    bool has_left = false;
    std::vector<double> Bhat;
    std::vector<double> b;
};

Problem generate_config(int32_t config, int32_t n);
void default_setup_options(amgcu_setup_options* so);
void default_solve_options(amgcu_solve_options* vo);
void config_options(int32_t c, amgcu_setup_options* so, amgcu_solve_options* vo);

}  // namespace amgcu
