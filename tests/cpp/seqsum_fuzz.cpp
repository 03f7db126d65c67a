// Host emulation of the exact sequential-order summation kernel (csrc/seqsum.cu)
// built on the same arithmetic core (csrc/seqsum.cuh): thread simulation, block tree
// merge, tile lists, group merges, final pass -- checked bit for bit against the
// reference's loop `double s = 0.0; for (i) s += t[i];` (sparse.hpp:309-313) on
// adversarial sequences.  Run by tests/test_seqsum_core.py (no GPU needed).
//
// usage: seqsum_fuzz <cases> <seed>   -> prints "ok <cases> <fallback_elems>" or the first mismatch
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_1610_03154_b200/csrc/seqsum.cuh"

using namespace amgcu::ss;

struct Geo {
    int threads, ipt, cap, tcap, tiles_per_group, gcap, pool;
};

static int64_t g_term_calls = 0;  // elements re-simulated (cost of the sequential merge steps)
struct Term {
    const std::vector<double>* t;
    double operator()(int64_t i) const {
        ++g_term_calls;
        return (*t)[static_cast<size_t>(i)];
    }
};

// tree merge of m lists laid out in pool at (off[j], len[j]), adjacent and ascending
static int tree_merge(Item* pool, std::vector<int>& off, std::vector<int>& len, const Term& term) {
    const int m = static_cast<int>(off.size());
    for (int step = 1; step < m; step <<= 1)
        for (int j = 0; j + step < m; j += 2 * step) len[j] = merge_pair(pool, off[j], len[j], off[j + step], len[j + step], term);
    return m ? len[0] : 0;
}

// merge a sequence of lists (each given as a vector) into one, through a bounded pool
static std::vector<Item> merge_lists(const std::vector<std::vector<Item>>& lists, int pool_cap, int acc_cap,
                                     const Term& term) {
    std::vector<Item> pool(static_cast<size_t>(pool_cap));
    int acc = 0;
    size_t idx = 0;
    while (idx < lists.size()) {
        std::vector<int> off, len;
        int at = acc;
        while (idx < lists.size() && at + static_cast<int>(lists[idx].size()) <= pool_cap && off.size() < 256) {
            for (size_t k = 0; k < lists[idx].size(); ++k) pool[at + k] = lists[idx][k];
            off.push_back(at);
            len.push_back(static_cast<int>(lists[idx].size()));
            at += static_cast<int>(lists[idx].size());
            ++idx;
        }
        if (off.empty()) {
            std::fprintf(stderr, "pool too small: acc %d next %zu cap %d\n", acc, lists[idx].size(), pool_cap);
            std::exit(2);
        }
        const int l0 = tree_merge(pool.data(), off, len, term);
        acc = merge_pair(pool.data(), 0, acc, off[0], l0, term);
        acc = truncate(pool.data(), acc, acc_cap);
    }
    return std::vector<Item>(pool.begin(), pool.begin() + acc);
}

// perturb: 0 = the kernel's approximations, 1 = garbage representatives (exercises the
// validation and fallback paths), 2 = zero tolerance
static double emulate(const std::vector<double>& t, const Geo& g, int perturb, std::mt19937_64& rng,
                      int64_t* fallback) {
    const int64_t n = static_cast<int64_t>(t.size());
    Term term{&t};
    if (n == 0) return 0.0;
    const int64_t tile = static_cast<int64_t>(g.threads) * g.ipt;
    const int64_t ntiles = (n + tile - 1) / tile;
    std::vector<std::vector<Item>> tile_lists;
    double P = 0.0, A = 0.0;  // approximate prefix (sum, abs sum) over previous tiles
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    for (int64_t T = 0; T < ntiles; ++T) {
        const int64_t base = T * tile;
        std::vector<double> ts(g.threads), ta(g.threads);
        for (int k = 0; k < g.threads; ++k) {
            double s = 0.0, a = 0.0;
            for (int j = 0; j < g.ipt; ++j) {
                const int64_t i = base + static_cast<int64_t>(k) * g.ipt + j;
                if (i < n) {
                    s += t[i];
                    a += std::fabs(t[i]);
                }
            }
            ts[k] = s;
            ta[k] = a;
        }
        // exclusive scan in a tree-ish order (different from the sequential chain)
        std::vector<double> es(g.threads), ea(g.threads);
        double cs = 0.0, ca = 0.0;
        for (int k = 0; k < g.threads; ++k) {
            es[k] = cs;
            ea[k] = ca;
            cs += ts[k];
            ca += ta[k];
        }
        // thread regions as in the kernel: cap items plus one 8-byte pad word
        const size_t region = static_cast<size_t>(g.cap) * sizeof(Item) + 8;
        std::vector<double> buf(static_cast<size_t>(g.threads) * region / 8 + 8);
        auto reg = [&](int k) { return reinterpret_cast<Item*>(reinterpret_cast<char*>(buf.data()) + k * region); };
        std::vector<int> off(g.threads), len(g.threads);
        for (int k = 0; k < g.threads; ++k) {
            const int64_t i0 = std::min<int64_t>(n, base + static_cast<int64_t>(k) * g.ipt);
            const int64_t i1 = std::min<int64_t>(n, i0 + g.ipt);
            double rep = P + es[k];
            double tau = std::ldexp(A + ea[k] + ta[k], -36);
            if (perturb == 1) {
                const int mode = static_cast<int>(rng() % 4);
                if (mode == 0) rep = rep * (1.0 + 1e-3 * U(rng));
                if (mode == 1) rep = -rep;
                if (mode == 2) rep = U(rng);
            }
            if (perturb == 2) tau = 0.0;
            Out o{reg(k), 0, g.cap};
            if (i1 > i0) simulate(o, rep, perturb == 0 && i0 == 0, i0, i1, tau, term);
            len[k] = o.n;
        }
        for (int step = 1; step < g.threads; step <<= 1)
            for (int j = 0; j + step < g.threads; j += 2 * step)
                len[j] = merge_ptr(reg(j), len[j], reg(j + step), len[j + step], term);
        const int L = truncate(reg(0), len[0], g.tcap);
        std::vector<Item> tl(reg(0), reg(0) + L);
        tile_lists.push_back(tl);
        P += cs;
        A += ca;
    }
    // groups
    const int64_t calls_tiles = g_term_calls;
    std::vector<std::vector<Item>> group_lists;
    for (size_t g0 = 0; g0 < tile_lists.size(); g0 += g.tiles_per_group) {
        std::vector<std::vector<Item>> part(tile_lists.begin() + g0,
                                            tile_lists.begin() + std::min(tile_lists.size(), g0 + g.tiles_per_group));
        group_lists.push_back(merge_lists(part, g.pool, g.gcap, term));
        if (std::getenv("SS_STATS") && g0 == 0) {
        }
    }
    const int64_t calls_groups = g_term_calls;
    std::vector<Item> fin = merge_lists(group_lists, g.pool, g.pool / 2, term);
    const int64_t calls_final = g_term_calls;
    if (std::getenv("SS_STATS")) {
        int64_t raw = 0, pieces = 0, tl = 0;
        for (auto& it : fin) {
            if (it.kind == kRaw) raw += it.i1 - it.i0; else ++pieces;
        }
        for (auto& l : tile_lists) tl += static_cast<int64_t>(l.size());
        int64_t gi = 0;
        for (auto& l : group_lists) gi += static_cast<int64_t>(l.size());
        std::printf("  n %lld tiles %lld tile-items %lld group-items %lld final items %zu raw %lld | resim group %lld final %lld\n",
                    static_cast<long long>(n), static_cast<long long>(ntiles), static_cast<long long>(tl),
                    static_cast<long long>(gi), fin.size(), static_cast<long long>(raw),
                    static_cast<long long>(calls_groups - calls_tiles), static_cast<long long>(calls_final - calls_groups));
    }
    return apply(fin.data(), static_cast<int>(fin.size()), 0.0, term, fallback);
}

static double seqsum(const std::vector<double>& t) {
    double s = 0.0;
    for (double v : t) s += v;
    return s;
}

static std::vector<double> gen(int kind, size_t n, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::normal_distribution<double> N(0.0, 1.0);
    std::vector<double> t(n);
    switch (kind) {
        case 0:  // random walk
            for (auto& v : t) v = U(rng);
            break;
        case 1:  // positive (monotone growth)
            for (auto& v : t) v = std::fabs(U(rng)) * 1e-3;
            break;
        case 2:  // walk with drift
            for (auto& v : t) v = U(rng) + 0.01;
            break;
        case 3: {  // products of two random vectors, one orthogonalised (final sum ~ 0)
            std::vector<double> x(n), y(n);
            for (size_t i = 0; i < n; ++i) {
                x[i] = 1.0 + 0.5 * U(rng);
                y[i] = U(rng);
            }
            double xy = 0, xx = 0;
            for (size_t i = 0; i < n; ++i) {
                xy += x[i] * y[i];
                xx += x[i] * x[i];
            }
            for (size_t i = 0; i < n; ++i) y[i] -= (xy / xx) * x[i];
            for (size_t i = 0; i < n; ++i) t[i] = x[i] * y[i];
            break;
        }
        case 4:  // exact cancellations: pairs v, -v, returning to exactly zero
            for (size_t i = 0; i + 1 < n; i += 2) {
                t[i] = U(rng);
                t[i + 1] = -t[i];
            }
            break;
        case 5:  // integer and half-integer terms at large magnitude: rounding ties
            for (auto& v : t) v = std::ldexp(static_cast<double>(static_cast<int64_t>(rng() % 7) - 3), 50) +
                                  (rng() % 2 ? 0.5 : -1.5);
            break;
        case 6:  // huge dynamic range, including extreme exponents
            for (auto& v : t) {
                const int e = static_cast<int>(rng() % 200) - 100;
                v = U(rng) * std::ldexp(1.0, e);
                if (rng() % 97 == 0) v = U(rng) * 1e300;
                if (rng() % 89 == 0) v = U(rng) * 1e-300;
            }
            break;
        case 7:  // zeros, signed zeros and a few specials
            for (auto& v : t) {
                const int r = static_cast<int>(rng() % 10);
                v = r < 5 ? 0.0 : (r < 7 ? -0.0 : U(rng));
            }
            if (n > 10 && rng() % 3 == 0) t[rng() % n] = (rng() % 2) ? INFINITY : NAN;
            break;
        case 8:  // constant terms (systematic rounding drift)
            for (auto& v : t) v = 0.1;
            break;
        case 9:  // sparse spikes in a sea of tiny values
            for (auto& v : t) v = (rng() % 1000 == 0) ? 1e8 * U(rng) : 1e-8 * U(rng);
            break;
        case 10:  // Gaussian walk scaled to 1e-6 with an occasional sign-flipping jump
            for (auto& v : t) v = 1e-6 * N(rng) + ((rng() % 5000 == 0) ? 1e-2 * U(rng) : 0.0);
            break;
        default:  // squares (norms)
            for (auto& v : t) {
                const double x = U(rng);
                v = x * x;
            }
    }
    return t;
}

static bool same(double a, double b) {
    if (std::isnan(a) && std::isnan(b)) return true;
    uint64_t x, y;
    std::memcpy(&x, &a, 8);
    std::memcpy(&y, &b, 8);
    return x == y;
}

int main(int argc, char** argv) {
    if (argc > 3) {  // stats mode: seqsum_fuzz 0 <seed> <n>
        std::mt19937_64 rng(1);
        const Geo g{256, 16, 4, 16, 256, 64, 1536};
        for (int kind = 0; kind < 12; ++kind) {
            auto t = gen(kind, std::strtoull(argv[3], nullptr, 10), rng);
            int64_t fb = 0;
            std::printf("kind %d\n", kind);
            const double got = emulate(t, g, 0, rng, &fb);
            std::printf("  %s fallback %lld\n", same(got, seqsum(t)) ? "ok" : "MISMATCH", static_cast<long long>(fb));
        }
        return 0;
    }
    const int cases = argc > 1 ? std::atoi(argv[1]) : 200;
    std::mt19937_64 rng(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
    const Geo geos[] = {{256, 16, 4, 16, 256, 64, 1536},  // the kernel's geometry
                        {8, 4, 3, 4, 3, 6, 64},             // tiny geometries: every level exercised
                        {4, 2, 2, 2, 2, 3, 16}};
    const size_t sizes[] = {0, 1, 2, 3, 17, 64, 255, 4095, 4096, 4097, 20000, 150000};
    int64_t fb_total = 0;
    for (int c = 0; c < cases; ++c) {
        const int kind = static_cast<int>(rng() % 12);
        const size_t n = sizes[rng() % (sizeof(sizes) / sizeof(sizes[0]))];
        const Geo& g = geos[rng() % 3];
        const int perturb = static_cast<int>(rng() % 5 == 0 ? 1 + rng() % 2 : 0);
        auto t = gen(kind, n, rng);
        int64_t fb = 0;
        const double got = emulate(t, g, perturb, rng, &fb);
        const double want = seqsum(t);
        if (perturb == 0) fb_total += fb;
        if (perturb == 0 && fb && std::getenv("SS_FB")) std::printf("fallback %lld: kind %d n %zu geo %d\n", (long long)fb, kind, n, g.threads);
        if (!same(got, want)) {
            std::printf("MISMATCH case %d kind %d n %zu geo %d/%d perturb %d: got %.17g want %.17g\n", c, kind, n,
                        g.threads, g.ipt, perturb, got, want);
            return 1;
        }
    }
    std::printf("ok %d %" PRId64 "\n", cases, fb_total);
    return 0;
}
