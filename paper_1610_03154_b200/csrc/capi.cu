// extern "C" boundary of libamgcu (include/amgcu.h).  Exceptions of the
// reference's types are mapped to status codes here; messages go to
// amgcu_last_error().
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "hier.cuh"
#include "small_dense.h"

using namespace amgcu;

struct amgcu_ctx_s {
    Ctx c;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
};

struct amgcu_hier_s {
    amgcu_ctx_s* owner;
    std::unique_ptr<DHier> h;
};

namespace {

thread_local std::string g_create_error;

template <typename F>
amgcu_status guarded(amgcu_ctx ctx, F&& f) {
    std::string* err = ctx ? &ctx->c.err : &g_create_error;
    try {
        f();
        return AMGCU_OK;
    } catch (const std::invalid_argument& e) {
        *err = e.what();
        return AMGCU_INVALID_ARGUMENT;
    } catch (const CudaFailure& e) {
        *err = e.what();
        return AMGCU_CUDA_ERROR;
    } catch (const std::runtime_error& e) {
        *err = e.what();
        return AMGCU_RUNTIME_ERROR;
    } catch (const std::logic_error& e) {
        *err = e.what();
        return AMGCU_LOGIC_ERROR;
    } catch (const std::exception& e) {
        *err = e.what();
        return AMGCU_INTERNAL;
    }
}

void check_csr(const amgcu_csr* m, const char* who) {
    if (!m || m->n_rows < 0 || m->n_cols < 0 || !m->row_offsets)
        throw InvalidArgument(std::string(who) + ": invalid CSR argument");
}

void up(Ctx& c, const amgcu_csr* m, DCsr& d) {
    check_csr(m, "amgcu");
    upload_csr(c, *m, d);
    sync(c);
}

void out_csr(const HostCsr& h, amgcu_csr* o) {
    o->n_rows = h.n_rows;
    o->n_cols = h.n_cols;
    o->nnz = h.nnz();
    o->block_size = h.block_size;
    o->row_offsets = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (h.n_rows + 1)));
    o->col_indices = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max(1, h.nnz())));
    o->values = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, h.nnz())));
    std::memcpy(o->row_offsets, h.row_offsets.data(), sizeof(int32_t) * (h.n_rows + 1));
    if (h.nnz()) {
        std::memcpy(o->col_indices, h.col_indices.data(), sizeof(int32_t) * h.nnz());
        std::memcpy(o->values, h.values.data(), sizeof(double) * h.nnz());
    }
}

void down(Ctx& c, const DCsr& d, amgcu_csr* o) { out_csr(download_csr(c, d), o); }

DBuf<double> up_vec(Ctx& c, const double* h, int64_t n) {
    DBuf<double> d(static_cast<size_t>(n), c.s);
    copy_h2d(c, d.get(), h, n);
    return d;
}

void down_vec(Ctx& c, double* h, const double* d, int64_t n) {
    copy_d2h(c, h, d, n);
    sync(c);
}

amgcu_hier make_hier(amgcu_ctx ctx, std::unique_ptr<DHier> h) {
    auto* out = new amgcu_hier_s;
    out->owner = ctx;
    out->h = std::move(h);
    return out;
}

void fill_report(const SolveResult& r, amgcu_solve_report* rep, double* history, int32_t cap) {
    if (rep) {
        rep->iterations = r.iterations;
        rep->converged = r.converged;
        rep->diverged = r.diverged;
        rep->history_len = static_cast<int32_t>(r.history.size());
        rep->rho = r.rho;
        rep->chi_oc = r.chi_oc;
        rep->chi_cc = r.chi_cc;
        rep->work_units_solve = r.wu_solve;
        rep->work_units_setup = r.wu_setup;
    }
    if (history)
        for (int32_t i = 0; i < cap && i < static_cast<int32_t>(r.history.size()); ++i) history[i] = r.history[i];
}

}  // namespace

extern "C" {

amgcu_status amgcu_ctx_create(int device, amgcu_ctx* out) {
    return guarded(nullptr, [&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw CudaFailure("amgcu_ctx_create: no CUDA device visible");
        }
        if (device < 0 || device >= count) throw InvalidArgument("amgcu_ctx_create: device out of range");
        AMG_CK(cudaSetDevice(device));
        auto* ctx = new amgcu_ctx_s;
        ctx->c.device = device;
        // the main stream gets the highest priority and the side stream (background work:
        // the evolution-SOC ledger count) the lowest, so the block scheduler fills idle SMs
        // with side work without delaying the main stream's kernels
        int prio_lo = 0, prio_hi = 0;
        AMG_CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        AMG_CK(cudaStreamCreateWithPriority(&ctx->c.s, cudaStreamNonBlocking, prio_hi));
        AMG_CK(cudaStreamCreateWithPriority(&ctx->c.side, cudaStreamNonBlocking, prio_lo));
        AMG_CK(cudaStreamCreateWithPriority(&ctx->c.side2, cudaStreamNonBlocking, prio_hi));
        ctx->c.main_s = ctx->c.s;
        AMG_CK(cudaDeviceGetAttribute(&ctx->c.sms, cudaDevAttrMultiProcessorCount, device));
        cudaMemPool_t pool;
        AMG_CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        AMG_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        *out = ctx;
    });
}

amgcu_status amgcu_ctx_destroy(amgcu_ctx ctx) {
    if (!ctx) return AMGCU_OK;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.s);
    ctx->c.scal.release();
    ctx->c.partials.release();
    ctx->c.tickets.release();
    ctx->c.arnoldi_v0.release();
    for (auto& w : ctx->c.ssws) {
        w.counters.release();
        w.status.release();
        w.lists.release();
        w.lens.release();
    }
    ctx->c.scan_tmp.release();  // every stream-ordered buffer before its stream goes
    cudaStreamSynchronize(ctx->c.s);
    ctx->c.cusolver.reset();  // bound to the context stream
    if (ctx->c.pin) cudaFreeHost(ctx->c.pin);
    cudaStreamSynchronize(ctx->c.side);
    cudaStreamSynchronize(ctx->c.side2);
    cudaStreamDestroy(ctx->c.side);
    cudaStreamDestroy(ctx->c.side2);
    cudaStreamDestroy(ctx->c.s);
    delete ctx;
    return AMGCU_OK;
}

const char* amgcu_last_error(amgcu_ctx ctx) { return ctx ? ctx->c.err.c_str() : g_create_error.c_str(); }

amgcu_status amgcu_ctx_set_sequential_reductions(amgcu_ctx ctx, int on) {
    return guarded(ctx, [&] { ctx->c.seq = on != 0; });
}

amgcu_status amgcu_ctx_set_candidate_overlap(amgcu_ctx ctx, int on) {
    return guarded(ctx, [&] { ctx->c.cand_overlap = on != 0; });
}

amgcu_status amgcu_ctx_set_masked_band(amgcu_ctx ctx, int32_t min_rows) {
    return guarded(ctx, [&] { ctx->c.band_min_rows = min_rows; });
}

amgcu_status amgcu_ctx_masked_band_stats(amgcu_ctx ctx, int64_t* accepted, int64_t* refused, int32_t* last_fail) {
    return guarded(ctx, [&] {
        *accepted = ctx->c.band_accepted;
        *refused = ctx->c.band_refused;
        *last_fail = ctx->c.band_last_fail;
    });
}

amgcu_status amgcu_ctx_synchronize(amgcu_ctx ctx) {
    return guarded(ctx, [&] { sync(ctx->c); });
}

amgcu_status amgcu_ctx_launch_count(amgcu_ctx ctx, int64_t* launches) {
    return guarded(ctx, [&] { *launches = ctx->c.launches; });
}

amgcu_status amgcu_ctx_sync_count(amgcu_ctx ctx, int64_t* syncs) {
    return guarded(ctx, [&] { *syncs = ctx->c.syncs; });
}

amgcu_status amgcu_ctx_timer_start(amgcu_ctx ctx) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (!ctx->t0) AMG_CK(cudaEventCreate(&ctx->t0));
        if (!ctx->t1) AMG_CK(cudaEventCreate(&ctx->t1));
        AMG_CK(cudaEventRecord(ctx->t0, c.s));
    });
}

amgcu_status amgcu_ctx_timer_stop(amgcu_ctx ctx, double* ms) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        AMG_CK(cudaEventRecord(ctx->t1, c.s));
        AMG_CK(cudaEventSynchronize(ctx->t1));
        float f = 0.f;
        AMG_CK(cudaEventElapsedTime(&f, ctx->t0, ctx->t1));
        *ms = f;
    });
}

amgcu_status amgcu_ctx_set_profiling(amgcu_ctx ctx, int on) {
    return guarded(ctx, [&] { ctx->c.profile = on != 0; });
}

amgcu_status amgcu_ctx_set_profile_mask(amgcu_ctx ctx, uint32_t family_mask) {
    return guarded(ctx, [&] { ctx->c.prof_mask = family_mask; });
}

amgcu_status amgcu_ctx_profile_reset(amgcu_ctx ctx) {
    return guarded(ctx, [&] {
        prof_collect(ctx->c);
        for (auto& r : ctx->c.prof) {
            r.launches = 0;
            r.bytes = 0.0;
            r.ms = 0.0;
        }
    });
}

amgcu_status amgcu_ctx_profile_query(amgcu_ctx ctx, int32_t family, int64_t* launches, double* ms, double* bytes) {
    return guarded(ctx, [&] {
        if (family < 0 || family >= kProfFamilies) throw InvalidArgument("profile family out of range");
        prof_collect(ctx->c);
        const ProfRecord& r = ctx->c.prof[family];
        *launches = r.launches;
        *ms = r.ms;
        *bytes = r.bytes;
    });
}

int32_t amgcu_profile_family_count(void) { return kProfFamilies; }

const char* amgcu_profile_family_name(int32_t family) {
    static const char* names[kProfFamilies] = {"vcycle_relax0_residual", "vcycle_restrict", "vcycle_prolong",
                                               "vcycle_post_relax",      "krylov_spmv",     "emin_masked_product",
                                               "spgemm",                 "evolution_soc",   "gauss_seidel_wavefront",
                                               "aggregate_lfmis",        "coarse_solve",    "blas1",
                                               "spectral_spmv",          "emin_cg",         "other",
                                               "arnoldi_blas1",          "emin_blas1",      "vcycle_coarse_fused"};
    return (family >= 0 && family < kProfFamilies) ? names[family] : "";
}

void amgcu_free(void* p) { std::free(p); }
void amgcu_csr_free(amgcu_csr* m) {
    if (!m) return;
    std::free(m->row_offsets);
    std::free(m->col_indices);
    std::free(m->values);
    m->row_offsets = nullptr;
    m->col_indices = nullptr;
    m->values = nullptr;
}

amgcu_status amgcu_setup(amgcu_ctx ctx, const amgcu_csr* A, int32_t k, const double* B, const double* left,
                         const amgcu_setup_options* opts, amgcu_hier* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        AMG_CK(cudaSetDevice(c.device));
        check_csr(A, "rn_setup");
        if (!B || !opts) throw InvalidArgument("rn_setup: null argument");
        DCsr dA;
        up(c, A, dA);
        const int64_t nk = static_cast<int64_t>(A->n_rows) * k;
        DBuf<double> dB = up_vec(c, B, nk);
        DBuf<double> dL;
        if (left) dL = up_vec(c, left, nk);
        *out = make_hier(ctx, rn_setup(c, dA, dB.get(), k, left ? dL.get() : nullptr, *opts));
    });
}

amgcu_status amgcu_setup_device(amgcu_ctx ctx, const amgcu_csr* A, int32_t k, const double* B, const double* left,
                                const amgcu_setup_options* opts, amgcu_hier* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        AMG_CK(cudaSetDevice(c.device));
        check_csr(A, "rn_setup");
        // wrap the caller's device arrays without copying: rn_setup clones A
        DCsr view;
        view.nr = A->n_rows;
        view.nc = A->n_cols;
        view.bs = A->block_size;
        view.nnz = A->nnz;
        // non-owning: build a temporary owning copy (clone keeps the API simple)
        view.rp.alloc(static_cast<size_t>(A->n_rows) + 1, c.s);
        view.ci.alloc(static_cast<size_t>(A->nnz), c.s);
        view.va.alloc(static_cast<size_t>(A->nnz), c.s);
        copy_d2d(c, view.rp.get(), A->row_offsets, A->n_rows + 1);
        copy_d2d(c, view.ci.get(), A->col_indices, A->nnz);
        copy_d2d(c, view.va.get(), A->values, A->nnz);
        static const bool ht = std::getenv("AMGCU_HOST_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        auto hh = rn_setup(c, view, B, k, left, *opts);
        const auto t1 = std::chrono::steady_clock::now();
        *out = make_hier(ctx, std::move(hh));
        if (ht)
            std::fprintf(stderr, "[host] rn_setup %.3f ms, returned after %.3f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    });
}

amgcu_status amgcu_hier_destroy(amgcu_hier h) {
    if (!h) return AMGCU_OK;
    amgcu_ctx ctx = h->owner;
    cudaSetDevice(ctx->c.device);
    h->h.reset();
    cudaStreamSynchronize(ctx->c.s);
    delete h;
    return AMGCU_OK;
}

amgcu_status amgcu_hier_levels(amgcu_hier h, int32_t* n_levels, int32_t* stagnated) {
    return guarded(h->owner, [&] {
        *n_levels = static_cast<int32_t>(h->h->lv.size());
        *stagnated = h->h->stagnated ? 1 : 0;
    });
}

amgcu_status amgcu_hier_get_matrix(amgcu_hier h, int32_t level, int32_t which, amgcu_csr* out) {
    return guarded(h->owner, [&] {
        if (level < 0 || level >= static_cast<int32_t>(h->h->lv.size())) throw InvalidArgument("level out of range");
        const DLevel& L = h->h->lv[level];
        const DCsr& M = which == 0 ? L.A : (which == 1 ? L.P : L.R);
        down(h->owner->c, M, out);
    });
}

amgcu_status amgcu_hier_get_candidates(amgcu_hier h, int32_t level, int32_t which, int32_t* n, int32_t* k,
                                       double** data) {
    return guarded(h->owner, [&] {
        if (level < 0 || level >= static_cast<int32_t>(h->h->lv.size())) throw InvalidArgument("level out of range");
        const DLevel& L = h->h->lv[level];
        const DBuf<double>& v = which == 0 ? L.B : L.Bc;
        const int32_t kk = L.k;
        *k = kk;
        *n = static_cast<int32_t>(v.size() / std::max(1, kk));
        *data = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(1, v.size())));
        down_vec(h->owner->c, *data, v.get(), static_cast<int64_t>(v.size()));
    });
}

amgcu_status amgcu_hier_level_symmetric(amgcu_hier h, int32_t level, int32_t* symmetric) {
    return guarded(h->owner, [&] { *symmetric = h->h->lv.at(level).symmetric ? 1 : 0; });
}

amgcu_status amgcu_hier_relax_weights(amgcu_hier h, int32_t level, double* pre, double* post) {
    return guarded(h->owner, [&] {
        const DLevel& L = h->h->lv.at(level);
        *pre = L.w_pre;
        *post = L.w_post;
    });
}

amgcu_status amgcu_hier_complexity(amgcu_hier h, double* chi_oc, double* chi_cc) {
    return guarded(h->owner, [&] {
        *chi_oc = operator_complexity(*h->h);
        *chi_cc = cycle_complexity(*h->h);
    });
}

amgcu_status amgcu_hier_ledger(amgcu_hier h, double* wu5) {
    return guarded(h->owner, [&] {
        Ctx& c = h->owner->c;
        AMG_CK(cudaSetDevice(c.device));
        double wu[5];
        hier_ledger(*h->h, wu);
        for (int b2 = 0; b2 < 5; ++b2) wu5[b2] = wu[b2];
    });
}

amgcu_status amgcu_solve(amgcu_hier h, const double* b, double* x, const amgcu_solve_options* opts,
                         amgcu_solve_report* report, double* history, int32_t history_cap) {
    return guarded(h->owner, [&] {
        Ctx& c = h->owner->c;
        AMG_CK(cudaSetDevice(c.device));
        const int32_t n = h->h->lv.front().A.nr;
        DBuf<double> db = up_vec(c, b, n);
        DBuf<double> dx = up_vec(c, x, n);
        SolveResult r = solve(*h->h, db.get(), dx.get(), *opts);
        down_vec(c, x, dx.get(), n);
        fill_report(r, report, history, history_cap);
    });
}

amgcu_status amgcu_solve_device(amgcu_hier h, const double* b_dev, double* x_dev, const amgcu_solve_options* opts,
                                amgcu_solve_report* report, double* history, int32_t history_cap) {
    return guarded(h->owner, [&] {
        AMG_CK(cudaSetDevice(h->owner->c.device));
        SolveResult r = solve(*h->h, b_dev, x_dev, *opts);
        fill_report(r, report, history, history_cap);
    });
}

amgcu_status amgcu_cycle(amgcu_hier h, double* x, const double* b, int32_t kind) {
    return guarded(h->owner, [&] {
        Ctx& c = h->owner->c;
        const int32_t n = h->h->lv.front().A.nr;
        DBuf<double> db = up_vec(c, b, n);
        DBuf<double> dx = up_vec(c, x, n);
        cycle(*h->h, dx.get(), db.get(), kind);
        down_vec(c, x, dx.get(), n);
    });
}

// ---- kernel-level entry points ----------------------------------------------------------
amgcu_status amgcu_spmv(amgcu_ctx ctx, const amgcu_csr* A, const double* x, double* y) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr d;
        up(c, A, d);
        DBuf<double> dx = up_vec(c, x, A->n_cols), dy(static_cast<size_t>(A->n_rows), c.s);
        spmv(c, d, dx.get(), dy.get());
        down_vec(c, y, dy.get(), A->n_rows);
    });
}

amgcu_status amgcu_dot(amgcu_ctx ctx, const double* x, const double* y, int64_t n, int32_t take_sqrt, double* out) {
    return guarded(ctx, [&] {
        if (n < 0) throw InvalidArgument("dot: negative length");
        Ctx& c = ctx->c;
        DBuf<double> dx = up_vec(c, x, n);
        DBuf<double> dy = take_sqrt ? DBuf<double>() : up_vec(c, y, n);
        DBuf<double> r(1, c.s);
        if (take_sqrt)
            nrm2(c, dx.get(), n, r.get());
        else
            dot(c, dx.get(), dy.get(), n, r.get());
        *out = read_scalar(c, r.get());
    });
}

amgcu_status amgcu_dot_device(amgcu_ctx ctx, const double* x_dev, const double* y_dev, int64_t n, int32_t take_sqrt,
                              double* out_dev) {
    return guarded(ctx, [&] {
        if (n < 0) throw InvalidArgument("dot: negative length");
        if (take_sqrt)
            nrm2(ctx->c, x_dev, n, out_dev);
        else
            dot(ctx->c, x_dev, y_dev, n, out_dev);
    });
}

amgcu_status amgcu_transpose(amgcu_ctx ctx, const amgcu_csr* A, amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr d, t;
        up(c, A, d);
        transpose(c, d, t);
        down(c, t, out);
    });
}

amgcu_status amgcu_matmul(amgcu_ctx ctx, const amgcu_csr* A, const amgcu_csr* B, amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr a, b, r;
        up(c, A, a);
        up(c, B, b);
        spgemm(c, a, b, r);
        down(c, r, out);
    });
}

amgcu_status amgcu_galerkin_product(amgcu_ctx ctx, const amgcu_csr* R, const amgcu_csr* A, const amgcu_csr* P,
                                    amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr r, a, p, o;
        up(c, R, r);
        up(c, A, a);
        up(c, P, p);
        galerkin(c, r, a, p, o);
        down(c, o, out);
    });
}

amgcu_status amgcu_filter_matrix(amgcu_ctx ctx, const amgcu_csr* G, int32_t theta_set, double theta, int32_t k,
                                 amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (k < 0) throw InvalidArgument("filter_matrix: k must be >= 1");
        DCsr g, f;
        up(c, G, g);
        filter_matrix(c, g, theta_set != 0, theta, k, f);
        down(c, f, out);
    });
}

amgcu_status amgcu_is_symmetric(amgcu_ctx ctx, const amgcu_csr* A, double tol, int32_t* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr a;
        up(c, A, a);
        *out = is_symmetric(c, a, tol) ? 1 : 0;
    });
}

amgcu_status amgcu_spectral_radius(amgcu_ctx ctx, const amgcu_csr* A, int32_t steps, double* rho) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr a;
        up(c, A, a);
        if (a.nr != a.nc) throw InvalidArgument("spectral_radius_estimate: square matrix required");
        if (a.nr == 0) {
            *rho = 0.0;
            return;
        }
        DBuf<double> dinv(static_cast<size_t>(a.nr), c.s);
        inverse_diagonal(c, a, dinv.get(), "spectral_radius_estimate: zero diagonal at row ");
        *rho = spectral_radius(c, a, steps, dinv.get());
    });
}

amgcu_status amgcu_strength(amgcu_ctx ctx, const amgcu_csr* A, const amgcu_strength_config* cfg, amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DLevel L;
        up(c, A, L.A);
        amgcu_setup_options o;
        default_setup_options(&o);
        o.strength_measure = cfg->measure;
        o.drop_tol = cfg->drop_tol;
        o.evolution_steps = cfg->evolution_steps;
        o.weighting = cfg->weighting;
        DCsr S;
        switch (cfg->measure) {
            case 0: classical_strength(c, L.A, cfg->drop_tol, S); break;
            case 1: symmetric_strength(c, L.A, cfg->drop_tol, S); break;
            case 2: {
                if (L.A.nr != L.A.nc) throw InvalidArgument("evolution_strength: square matrix required");
                if (cfg->drop_tol <= 0.0) throw InvalidArgument("evolution_strength: drop_tol must be positive");
                if (cfg->evolution_steps < 1) throw InvalidArgument("evolution_strength: steps must be >= 1");
                const int32_t n = L.A.nr;
                std::vector<double> winv(n);
                HostCsr h = download_csr(c, L.A);
                if (cfg->weighting == 0) {
                    const double rho = level_rho(c, L);
                    if (rho <= 0.0) throw RuntimeError("evolution_strength: spectral radius estimate failed");
                    const double omega = 1.0 / rho;
                    for (int32_t i = 0; i < n; ++i) {
                        double d = 0.0;
                        for (int32_t p = h.row_offsets[i]; p < h.row_offsets[i + 1]; ++p)
                            if (h.col_indices[p] == i) d = h.values[p];
                        if (d == 0.0)
                            throw RuntimeError("evolution_strength: zero diagonal at row " + std::to_string(i));
                        winv[i] = omega / d;
                    }
                } else {
                    for (int32_t i = 0; i < n; ++i) {
                        double s = 0.0;
                        for (int32_t p = h.row_offsets[i]; p < h.row_offsets[i + 1]; ++p) s += std::fabs(h.values[p]);
                        if (s == 0.0) throw RuntimeError("evolution_strength: zero row at " + std::to_string(i));
                        winv[i] = 1.0 / s;
                    }
                }
                DBuf<double> dw = up_vec(c, winv.data(), n);
                DCsr At;
                transpose(c, L.A, At);
                evolution_strength(c, L.A, At, dw.get(), cfg->drop_tol, cfg->evolution_steps, S);
                break;
            }
            default: throw InvalidArgument("strength: unknown measure");
        }
        down(c, S, out);
    });
}

amgcu_status amgcu_normalize_strength(amgcu_ctx ctx, const amgcu_csr* S, amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr s, n;
        up(c, S, s);
        normalize_strength(c, s, n);
        down(c, n, out);
    });
}

amgcu_status amgcu_amalgamate(amgcu_ctx ctx, const amgcu_csr* S, int32_t m, amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr s, n;
        up(c, S, s);
        amalgamate(c, s, m, n);
        down(c, n, out);
    });
}

amgcu_status amgcu_greedy_aggregate(amgcu_ctx ctx, const amgcu_csr* S, int32_t* n_agg, int32_t* node_to_agg,
                                    int32_t* roots) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DCsr s;
        up(c, S, s);
        DAgg agg;
        greedy_aggregate(c, s, agg);
        *n_agg = agg.n_agg;
        copy_d2h(c, node_to_agg, agg.owner.get(), agg.n_nodes);
        copy_d2h(c, roots, agg.roots.get(), agg.n_agg);
        sync(c);
    });
}

amgcu_status amgcu_sparsity_pattern(amgcu_ctx ctx, const amgcu_csr* S, const amgcu_csr* C, int32_t degree,
                                    amgcu_csr* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (S->n_rows != S->n_cols || S->n_cols != C->n_rows)
            throw InvalidArgument("sparsity_pattern: dimension mismatch");
        if (degree < 0) throw InvalidArgument("sparsity_pattern: degree must be >= 0");
        DCsr s, n;
        up(c, S, s);
        up(c, C, n);
        for (int t = 0; t < degree; ++t) {
            DCsr nx;
            spgemm(c, s, n, nx);
            n = std::move(nx);
        }
        n.bs = C->block_size;
        down(c, n, out);
    });
}

amgcu_status amgcu_improve_candidates(amgcu_ctx ctx, const amgcu_csr* A, int32_t k, const double* B,
                                      int32_t sweeps, int32_t scheme, double weight, double* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        DLevel L;
        up(c, A, L.A);
        if (L.A.nr != L.A.nc) throw InvalidArgument("improve_candidates: dimension mismatch");
        const int64_t nk = static_cast<int64_t>(A->n_rows) * k;
        DBuf<double> dB = up_vec(c, B, nk);
        improve_candidates(c, L.A, dB.get(), k, sweeps, scheme, weight, &L);
        down_vec(c, out, dB.get(), nk);
    });
}

amgcu_status amgcu_relax(amgcu_ctx ctx, const amgcu_csr* A, int32_t scheme, double weight, int32_t sweeps, double* x,
                         const double* b) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        require_supported_relax(scheme, "relax");
        DLevel L;
        up(c, A, L.A);
        if (L.A.nr != L.A.nc) throw InvalidArgument("relax: square matrix required");
        const int32_t n = L.A.nr;
        DBuf<double> dx = up_vec(c, x, n), db = up_vec(c, b, n);
        if (scheme == 3 || scheme == 4) {
            // relaxation.hpp:67-97, 128-167
            if (scheme == 3) {
                GsneWs ws;
                gsne_workspace(c, L.A, ws);
                gsne(c, L.A, ws, dx.get(), db.get(), sweeps);
            } else {
                DBuf<double> inv;
                block_workspace(c, L.A, inv);
                block_sym_gs(c, L.A, inv.get(), dx.get(), db.get(), sweeps);
            }
            down_vec(c, x, dx.get(), n);
            return;
        }
        L.inv_diag.alloc(static_cast<size_t>(n), c.s);
        inverse_diagonal(c, L.A, L.inv_diag.get(), "relax: zero diagonal at row ");
        if (scheme == 0) {
            const double w = weight != 0.0 ? weight : 4.0 / (3.0 * level_rho(c, L));
            std::vector<double> hd(n);
            copy_d2h(c, hd.data(), L.inv_diag.get(), n);
            sync(c);
            for (auto& v : hd) v = w * v;
            DBuf<double> wd = up_vec(c, hd.data(), n);
            jacobi(c, L.A, wd.get(), dx.get(), db.get(), 1, sweeps);
        } else {
            gauss_seidel(c, L.A, L.inv_diag.get(), dx.get(), db.get(), 1, sweeps, scheme == 2);
        }
        down_vec(c, x, dx.get(), n);
    });
}

amgcu_status amgcu_generate(int32_t config, int32_t n, amgcu_csr* A, int32_t* k, double** B, int32_t* has_left,
                            double** Bhat, double** b) {
    return guarded(nullptr, [&] {
        Problem p = generate_config(config, n);
        out_csr(p.A, A);
        *k = p.k;
        *B = static_cast<double*>(std::malloc(sizeof(double) * p.B.size()));
        std::memcpy(*B, p.B.data(), sizeof(double) * p.B.size());
        *has_left = p.has_left ? 1 : 0;
        *Bhat = nullptr;
        if (p.has_left) {
            *Bhat = static_cast<double*>(std::malloc(sizeof(double) * p.Bhat.size()));
            std::memcpy(*Bhat, p.Bhat.data(), sizeof(double) * p.Bhat.size());
        }
        *b = static_cast<double*>(std::malloc(sizeof(double) * p.b.size()));
        std::memcpy(*b, p.b.data(), sizeof(double) * p.b.size());
    });
}

amgcu_status amgcu_config_options(int32_t config, amgcu_setup_options* so, amgcu_solve_options* vo) {
    return guarded(nullptr, [&] { config_options(config, so, vo); });
}

void amgcu_default_setup_options(amgcu_setup_options* so) { default_setup_options(so); }
void amgcu_default_solve_options(amgcu_solve_options* vo) { default_solve_options(vo); }

}  // extern "C"
