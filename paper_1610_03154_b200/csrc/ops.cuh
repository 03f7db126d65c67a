// Declarations of the sm_100a kernel families of libamgcu (host launchers).
// Every launcher reproduces one reference routine with the reference's
// per-entry operation order (compiled with --fmad=false), so the integer
// structure it emits is bit-identical and the fp64 values are bit-identical
// given bit-identical inputs (SURVEY.md §7 hard part 1).
#pragma once

#include <memory>

#include "device.cuh"

namespace amgcu {

// ---- sparse core (sparse_core.cu) -----------------------------------------------------
// y = A x, sequential row sums in CSR order (sparse.hpp:141-152)
void spmv(Ctx& c, const DCsr& A, const double* x, double* y);
// transpose with rows ascending inside each column (sparse.hpp:161-179)
void transpose(Ctx& c, const DCsr& A, DCsr& T);
// positions of A's entries in transposed (CSC) order: colptr (nc+1), pos (nnz)
void transpose_positions(Ctx& c, const DCsr& A, DBuf<int32_t>& colptr, DBuf<int32_t>& pos, DBuf<int32_t>* src_row);
// C = A B, per-entry sums in A-row then B-row order, exact zeros dropped
// (sparse.hpp:183-217); *ops receives the multiply-model count.
void spgemm(Ctx& c, const DCsr& A, const DCsr& B, DCsr& C, double* ops = nullptr);
// R (A P) (sparse.hpp:220-228)
void galerkin(Ctx& c, const DCsr& R, const DCsr& A, const DCsr& P, DCsr& C, double* ops = nullptr);
// filter_matrix (sparse.hpp:236-272); k <= 0 means unset
void filter_matrix(Ctx& c, const DCsr& G, bool theta_set, double theta, int32_t k, DCsr& F);
// is_symmetric (sparse.hpp:288-305)
bool is_symmetric(Ctx& c, const DCsr& A, double tol);
// dinv[i] = 1 / A(i,i); throws RuntimeError(prefix + row) for the lowest zero diagonal
void inverse_diagonal(Ctx& c, const DCsr& A, double* dinv, const char* prefix);
// the same without the throw: the first zero-diagonal row, or -1
int32_t inverse_diagonal_check(Ctx& c, const DCsr& A, double* dinv);
void diagonal(Ctx& c, const DCsr& A, double* d);
// max_i |v_i| (exact)
double max_abs(Ctx& c, const double* v, int64_t n);
// drop entries with vals[p] == 0 from pattern N (from_pattern_values, interpolation.hpp:229-243)
void compact_pattern(Ctx& c, const DCsr& N, const double* vals, int32_t bs, DCsr& out);
// row index of every stored entry
void entry_rows(Ctx& c, const DCsr& A, int32_t* rows);

// ---- BLAS-1 with device-resident scalars (blas.cu) -----------------------------------
// *out = sum_i x_i y_i.  seq mode (default): the reference's order (sparse.hpp:309-313),
// bit for bit; otherwise a deterministic two-stage tree.
void dot(Ctx& c, const double* x, const double* y, int64_t n, double* out);
// *out = sqrt(dot(x, x))
void nrm2(Ctx& c, const double* x, int64_t n, double* out);
// x += st[2] p, r -= st[2] q, *out = ||r|| in one pass
bool pcg_update_nrm(Ctx& c, const double* st, const int32_t* bad, const double* p, const double* q, double* x,
                    double* r, int64_t n, double* out);
// y += s * x with s = sign * (*alpha)   (axpy, sparse.hpp:317-319)
void axpy_dev(Ctx& c, const double* alpha, double sign, const double* x, double* y, int64_t n);
// x *= 1 / (*denom)                      (scale(1.0 / h, v))
void scale_recip_dev(Ctx& c, const double* denom, double* x, int64_t n);
// y += sign * (*alpha) * x; *out = dot(y, z) (z null: dot(y, y), sqrt if take_sqrt) -- one pass
void axpy_dot(Ctx& c, const double* alpha, double sign, const double* x, double* y, const double* z, int64_t n,
              double* out, bool take_sqrt);
void scale_const(Ctx& c, double alpha, double* x, int64_t n);
// grid of the tree reductions for length n (the cooperative Arnoldi reproduces it)
unsigned dot_grid(Ctx& c, int64_t n);
// seqsum.cu: the same sums in the reference's exact order, one launch each
void seqsum_dot(Ctx& c, const double* x, const double* y, int64_t n, double* out, bool take_sqrt);
void seqsum_axpy_dot(Ctx& c, const double* alpha, double sign, const double* x, double* y, const double* z, int64_t n,
                     double* out, bool take_sqrt);
void seqsum_pcg_update_nrm(Ctx& c, const double* st, const int32_t* bad, const double* p, const double* q, double* x,
                           double* r, int64_t n, double* out);

// ---- strength / aggregation (strength.cu, aggregate.cu) --------------------------------
void symmetric_strength(Ctx& c, const DCsr& A, double theta, DCsr& S);
void classical_strength(Ctx& c, const DCsr& A, double theta, DCsr& S);
// evolution strength (strength.hpp:116-238); winv per row
void evolution_strength(Ctx& c, const DCsr& A, const DCsr& At, const double* winv, double drop_tol, int steps,
                        DCsr& S);
// WorkLedger count of evolution_strength on A (exact).  Started on the context's side
// stream right after the SOC (it reuses the SOC's transpose, kept here for the host
// fallback of large balls) so it overlaps the rest of the setup; collected by
// evolution_ops_finish.
struct EvoCount {
    DCsr At;
    DBuf<unsigned long long> total;
    DBuf<int32_t> ovf, novf;
    int steps = 0;
    cudaStream_t s = nullptr;     // stream the buffers are released on
    cudaEvent_t done = nullptr;   // recorded on the side stream after the count
    EvoCount() = default;
    EvoCount(const EvoCount&) = delete;
    EvoCount& operator=(const EvoCount&) = delete;
    ~EvoCount();
};
std::unique_ptr<EvoCount> evolution_ops_start(Ctx& c, const DCsr& A, DCsr&& At, int steps);
double evolution_ops_finish(Ctx& c, const DCsr& A, EvoCount& e);
void normalize_strength(Ctx& c, const DCsr& S, DCsr& N);
void amalgamate(Ctx& c, const DCsr& S, int32_t m, DCsr& N);
struct DAgg {
    int32_t n_nodes = 0, n_agg = 0;
    DBuf<int32_t> owner;  // node_to_agg
    DBuf<int32_t> roots;
};
void greedy_aggregate(Ctx& c, const DCsr& S, DAgg& agg);
void aggregate_indicator(Ctx& c, const DAgg& agg, DCsr& Cm);

// ---- spectral radius (arnoldi.cu) ----------------------------------------------------
// *built_out (optional) receives the Krylov dimension reached (the reference's SpMV count)
double spectral_radius(Ctx& c, const DCsr& A, int steps, const double* dinv, int* built_out = nullptr);
// the same in two halves: start queues the Arnoldi process and the copy of H on c.s (no
// host synchronisation: it may run on a side stream), finish waits and takes the
// eigenvalues.  The start vector must cover n first (ensure_start_vector, main stream).
struct ArnoldiJob {
    int32_t n = 0;
    int m = 0;
    DBuf<double> V, Hd;
    double* hpin = nullptr;
    cudaEvent_t done = nullptr;
    ArnoldiJob() = default;
    ArnoldiJob(const ArnoldiJob&) = delete;
    ArnoldiJob& operator=(const ArnoldiJob&) = delete;
    ~ArnoldiJob();
};
void ensure_start_vector(Ctx& c, size_t n);
std::unique_ptr<ArnoldiJob> spectral_radius_start(Ctx& c, const DCsr& A, int steps, const double* dinv);
double spectral_radius_finish(Ctx& c, ArnoldiJob& job, int* built_out);

// ---- relaxation (relax.cu) -----------------------------------------------------------
// sync-free wavefront Gauss-Seidel sweeps (relaxation.hpp:115-127) over k columns
// (column-major x of size n*k; b n*k or nullptr for b = 0)
// The lane-per-segment Gauss-Seidel kernel (gs_lanes.cuh) for forward sweeps: its plan
// for a matrix (segments, longest row; host synchronisations) and one column's sweeps
// (no host synchronisation: may run on another stream than the plan's)
constexpr int kGsMaxColumns = 8;  // candidate columns one Gauss-Seidel launch relaxes

struct LanePlan {  // the forward-sweep plan of a matrix (relax.cu: lane_plan)
    enum Kind { kNone = 0, kLanes = 1, kSegWarp = 2, kCta = 3 };
    bool ok = false;
    int kind = kNone;
    int32_t nf = 0, longest_row = 0;
    DBuf<int32_t> segf;
};
LanePlan lane_plan(Ctx& c, const DCsr& A, int nsw, int k);
// forward sweeps of the k columns of x (n x k column-major; b likewise, or null)
void gs_lanes_run(Ctx& c, const DCsr& A, const LanePlan& pl, const double* inv_diag, double* x, const double* b,
                  int nsw, int32_t k);

void gauss_seidel(Ctx& c, const DCsr& A, const double* inv_diag, double* x, const double* b, int k, int sweeps,
                  bool symmetric_sweep);
// weighted Jacobi sweeps x += (w dinv) (b - A x) (relaxation.hpp:107-113); b may be nullptr (0)
void jacobi(Ctx& c, const DCsr& A, const double* wdinv, double* x, const double* b, int k, int sweeps);

// relax_more.cu: gsne (relaxation.hpp:128-142) and block symmetric Gauss-Seidel
// (relaxation.hpp:143-167), one column of x; workspaces as make_relax_workspace
// (relaxation.hpp:67-97): A^T and the squared column norms / the diagonal block inverses
struct GsneWs {
    DCsr At;
    DBuf<double> cn2;
};
void gsne_workspace(Ctx& c, const DCsr& A, GsneWs& ws);
void gsne(Ctx& c, const DCsr& A, const GsneWs& ws, double* x, const double* b, int sweeps);
void block_workspace(Ctx& c, const DCsr& A, DBuf<double>& inv);
void block_sym_gs(Ctx& c, const DCsr& A, const double* inv, double* x, const double* b, int sweeps);

}  // namespace amgcu
