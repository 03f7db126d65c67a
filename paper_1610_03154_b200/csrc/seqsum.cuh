// Exact sequential-order summation, the arithmetic core (host + device).
//
// The reference sums every global reduction left to right from +0.0:
//     double s = 0.0; for (i) s += t[i];                    (sparse.hpp:309-313)
// and the hierarchy it builds depends on the last bits of those sums (the Arnoldi rho
// feeds the evolution-SOC thresholds, the energy-min CG dots feed P and through RAP the
// is_symmetric branch of every coarse level).  This header evaluates that exact
// left-to-right chain in parallel; csrc/seqsum.cu is the kernel around it and
// tests/cpp/seqsum_fuzz.cpp emulates the kernel on the host against the plain loop.
//
// Translation lemma.  Let v be real with |v| in [2^b, 2^(b+1)), and Delta an EVEN
// multiple of u_b = 2^(b-52) with v + Delta in the same signed binade.  Then
// RN(v + Delta) = RN(v) + Delta (the grid of the binade is the multiples of u_b, and an
// even shift keeps the ties-to-even choice).
//
// Piece.  Over elements [i0, i1), a piece holds two representative start states
// rep[0], rep[1] = rep[0] +- u_E, both in binade E (adjacent doubles, one of each
// mantissa parity), the states end[c] the chain reaches from rep[c] (simulated
// exactly, one DADD per element), and a window W.  Claim: for a true start s with
// |s - rep[0]| < W, let c be the parity of (s - rep[0]) / u_E; then the chain from s
// ends at end[c] + (s - rep[c]).  Proof: W never exceeds the distance of either rep to
// its binade edges, so s lies in binade E and Delta = s - rep[c] is an even multiple
// of u_E.  Every absorbed element's exact sum (in both chains) lies in a binade
// b <= E, so Delta is an even multiple of u_b as well, and W never exceeds that
// sum's distance to its binade edges (minus the u_E between the chains), so the
// shifted sum stays in binade b.  Induct with the lemma.
//
// Elements a piece cannot absorb (a sum rising above E, an exact zero, a sum closer
// to a binade edge than the tolerance tau, non-finite or extreme values) are *raw*:
// unresolved in the list, re-simulated when a piece to their left (whose state is
// closer to the true one) is merged with them.  The chain from +0.0 before element 0
// is known exactly (kExact: no window, absorbs everything), so the final merge sweeps
// every remaining raw element into it.  Pieces compose: L then R with L's ends inside
// R's window gives a piece with L's reps, R's ends shifted, and the window shrunk by
// the shift -- every operation exact.  The final pass applies the list to s = +0.0; a
// piece whose window does not hold the true state is summed element by element
// (correct, slow).  The result is always the reference's bits; the windows, the
// tolerance and the list capacities only decide the speed.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <climits>

#ifdef __CUDACC__
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD inline
#endif

namespace amgcu {
namespace ss {

enum : int32_t { kPiece = 0, kRaw = 1, kExact = 2 };

constexpr int kInline = 5;  // terms a raw item carries (re-simulation without reloading them)

struct Item {
    union {
        struct {
            double rep[2];  // piece: representative start states (parity classes); exact: rep[0]
            double end[2];  // piece: end states of the two chains; exact: end[0]
            double W;       // piece: strict validity window |s - rep[0]| < W
        };
        double tv[kInline];  // raw: the terms of its first E elements
    };
    double tau;      // tolerance below which a binade-edge distance makes an element raw
    int32_t i0, i1;  // element range [i0, i1) (sums of up to 2^31 - 1 terms)
    int32_t E;       // piece: binade of the representatives; raw: terms held inline
    int32_t kind;
};
static_assert(sizeof(Item) == 64, "8 words: list regions are padded to an odd word count");

// term of element i of raw item r (inline if held, else from the accessor); selects
// instead of an indexed load keep a register copy of r out of local memory
template <class TermAt>
SS_HD double raw_term(const Item& r, int64_t i, const TermAt& term) {
    const int64_t k = i - r.i0;
    if (k >= r.E) return term(i);
    static_assert(kInline == 5, "raw_term selects");
    return k == 0 ? r.tv[0] : k == 1 ? r.tv[1] : k == 2 ? r.tv[2] : k == 3 ? r.tv[3] : r.tv[4];
}

SS_HD uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
#endif
}
SS_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    std::memcpy(&x, &u, 8);
    return x;
#endif
}
// unbiased exponent of a finite non-zero double (subnormals report -1023)
SS_HD int32_t expo(double x) { return static_cast<int32_t>((bits(x) >> 52) & 0x7ff) - 1023; }
SS_HD double pow2(int32_t e) { return from_bits(static_cast<uint64_t>(e + 1023) << 52); }  // normal range only
SS_HD bool mantissa_zero(double x) { return (bits(x) & 0x000fffffffffffffull) == 0; }
// a lower bound of the exact a - b when that is positive: RN(a - b) stepped down one
// ulp (one integer decrement of the bits).  Non-positive results are returned as they
// are: every caller treats a non-positive window or slack as "not usable".
SS_HD double sub_down(double a, double b) {
    const double d = a - b;
    return d > 0.0 ? from_bits(bits(d) - 1) : d;
}
SS_HD double dmin(double a, double b) { return a < b ? a : b; }

constexpr int32_t kMinBinade = -960;  // keeps every quantity (down to u_b / 2) normal
constexpr int32_t kMaxBinade = 1000;

// distance of x (normal, binade e) to the edges of its binade; exact
SS_HD double edge_slack(double x, int32_t e) {
    const double a = std::fabs(x);
    return dmin(a - pow2(e), pow2(e + 1) - a);
}

// One chain step s -> RN(s + t).  Returns false when the exact sum is zero, non-finite,
// outside [kMinBinade, emax] or closer than tau to its binade edges; otherwise *h is
// the new state and *slack a lower bound of the exact sum's distance to its edges.
SS_HD bool step(double s, double t, int32_t emax, double tau, double* h_out, double* slack_out,
                bool* tie_at_emax = nullptr) {
    const double h = s + t;
    if (!(std::fabs(h) < INFINITY) || h == 0.0) return false;
    // TwoSum: the exact sum is h + l
    const double bb = h - s;
    const double l = (s - (h - bb)) + (t - bb);
    int32_t b = expo(h);
    const bool lopp = (l != 0.0) && ((l < 0.0) != (h < 0.0));
    const double al = std::fabs(l);
    double slack;
    if (mantissa_zero(h) && lopp) {
        // |h| = 2^e and the exact sum lies just below it: binade e - 1
        b -= 1;
        if (b < kMinBinade) return false;
        slack = dmin(sub_down(pow2(b), al), al);  // |v| - 2^b = 2^b - |l|,  2^(b+1) - |v| = |l|
    } else {
        if (b < kMinBinade) return false;
        const double ah = std::fabs(h);
        double lo = ah - pow2(b);      // exact (same binade)
        double hi = pow2(b + 1) - ah;  // exact
        if (l != 0.0) {
            if (lopp)
                lo = sub_down(lo, al);
            else
                hi = sub_down(hi, al);
        }
        slack = dmin(lo, hi);
    }
    if (b > emax) return false;
    if (!(slack > 0.0) || slack < tau) return false;
    *h_out = h;
    *slack_out = slack;
    // a rounding tie: the exact sum halfway between two doubles of binade b
    if (tie_at_emax) *tie_at_emax = b == emax && al == pow2(b - 53);
    return true;
}

SS_HD void open_exact(double rep, double tau, int64_t i0, Item& p);

// Open a piece at (approximate) state rep before element i0.  A zero state opens an
// exact-match piece at +0.0 (the running sum is never -0.0: it starts at +0.0 and an
// exact cancellation rounds to +0.0), which applies when the true state is +0.0 --
// runs of zero terms and exact cancellations.
SS_HD bool open_piece(double rep, double tau, int64_t i0, Item& p) {
    if (rep == 0.0) {
        open_exact(0.0, tau, i0, p);
        return true;
    }
    if (!(std::fabs(rep) < INFINITY)) return false;
    const int32_t e = expo(rep);
    if (e < kMinBinade || e > kMaxBinade) return false;
    // the other parity class: the adjacent double inside the binade
    const double u = pow2(e - 52);
    const double sg = rep < 0.0 ? -1.0 : 1.0;
    double r1 = rep + sg * u;
    if (expo(r1) != e) r1 = rep - sg * u;
    const double w = dmin(edge_slack(rep, e), edge_slack(r1, e));
    if (!(w > u) || w < tau) return false;
    p.rep[0] = p.end[0] = rep;
    p.rep[1] = p.end[1] = r1;
    p.W = w;
    p.tau = tau;
    p.i0 = p.i1 = static_cast<int32_t>(i0);
    p.E = e;
    p.kind = kPiece;
    return true;
}

SS_HD void open_exact(double rep, double tau, int64_t i0, Item& p) {
    p.rep[0] = p.end[0] = rep;
    p.rep[1] = p.end[1] = rep;
    p.W = 0.0;
    p.tau = tau;
    p.i0 = p.i1 = static_cast<int32_t>(i0);
    p.E = 0;
    p.kind = kExact;
}

// Try to absorb element p.i1 (term t) into piece p.
SS_HD bool absorb(Item& p, double t) {
    if (p.kind == kExact) {
        p.end[0] = p.end[0] + t;
        p.i1 += 1;
        return true;
    }
    // Chain 1 is chain 0 shifted by off = end[1] - end[0] (exact: adjacent doubles, a
    // multiple of u_E of size <= 2 u_E).  By the lemma the shift carries through every
    // step whose sum stays in its binade, except a tie at binade E while off is an odd
    // multiple of u_E: only then is chain 1 stepped on its own.
    double h0, s0;
    bool tie = false;
    if (!step(p.end[0], t, p.E, p.tau, &h0, &s0, &tie)) return false;
    const double u = pow2(p.E - 52);
    const double off = p.end[1] - p.end[0];
    const double aoff = std::fabs(off);
    double h1;
    double w = dmin(p.W, sub_down(s0, aoff + u));  // chain 1's sum is within |off| of chain 0's
    if (tie && aoff == u) {
        double s1;
        if (!step(p.end[1], t, p.E, p.tau, &h1, &s1)) return false;
        w = dmin(w, sub_down(s1, u));
    } else {
        h1 = h0 + off;  // the true state of chain 1: representable, so exact
    }
    // a start within W of rep[0] lies within W + u_E of rep[1]
    if (!(w > 0.0) || w < p.tau) return false;
    p.W = w;
    p.end[0] = h0;
    p.end[1] = h1;
    p.i1 += 1;
    return true;
}

// parity of d / u_e for d an exact multiple of u_e with |d| < 2^(e+1)
SS_HD int parity_units(double d, int32_t e) {
    const double k = d * pow2(52 - e);  // an exact integer, |k| < 2^53
    const long long ik = static_cast<long long>(k);
    return static_cast<int>(ik & 1ll);
}

// Compose piece L with the piece R that follows it; false (L unchanged) if R's window
// does not hold L's end states.
SS_HD bool compose(Item& L, const Item& R) {
    if (R.kind == kExact) {  // only L exact with the same state can continue it
        if (L.kind != kExact || bits(L.end[0]) != bits(R.rep[0])) return false;
        L.end[0] = L.end[1] = R.end[0];
        L.i1 = R.i1;
        return true;
    }
    if (R.kind != kPiece) return false;
    // the offsets of L's valid starts are even multiples of u_{E_L}; R's parity rule
    // needs them to be even multiples of u_{E_R}
    if (L.kind == kPiece && R.E > L.E) return false;
    const int nch = L.kind == kExact ? 1 : 2;
    double ne[2] = {0.0, 0.0}, shrink = 0.0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        if (c >= nch) break;
        const double le = c ? L.end[1] : L.end[0];
        const double d0 = le - R.rep[0];  // exact whenever |d0| < R.W (same binade)
        if (!(std::fabs(d0) < R.W)) return false;
        const int q = parity_units(d0, R.E);
        const double d = q ? le - R.rep[1] : d0;  // exact: same binade
        ne[c] = (q ? R.end[1] : R.end[0]) + d;    // chain c's true state: representable, so exact
        if (std::fabs(d0) > shrink) shrink = std::fabs(d0);
    }
    if (L.kind == kPiece) {
        // a start rep_c + Delta (|Delta| < L.W + u_{E_L}) ends L at end_c + Delta; R
        // holds it when |end_c - R.rep[0] + Delta| < R.W
        const double w = dmin(L.W, sub_down(sub_down(R.W, shrink), pow2(L.E - 52)));
        if (!(w > 0.0)) return false;
        L.W = w;
    }
    L.end[0] = ne[0];
    L.end[1] = nch == 2 ? ne[1] : ne[0];
    L.i1 = R.i1;
    return true;
}

// Output cursor over an item array (a list being built in place).
struct Out {
    Item* a;
    int n;    // items written
    int cap;  // slots that may be written: a[0 .. cap)
    SS_HD Item& last() { return a[n - 1]; }
    // raw element i (term t) after the items
    SS_HD void push_raw1(int64_t i, double t, double tau) {
        if (n > 0 && a[n - 1].kind == kRaw && a[n - 1].i1 == i) {
            Item& r = a[n - 1];
            if (r.E == i - r.i0 && r.E < kInline) r.tv[r.E++] = t;
            r.i1 = static_cast<int32_t>(i + 1);
            return;
        }
        Item& r = a[n++];
        r.kind = kRaw;
        r.i0 = static_cast<int32_t>(i);
        r.i1 = static_cast<int32_t>(i + 1);
        r.tau = tau;
        r.tv[0] = t;
        r.E = 1;
    }
    // raw range [i0, i1) without its terms
    SS_HD void push_raw(int64_t i0, int64_t i1, double tau) {
        if (n > 0 && a[n - 1].kind == kRaw && a[n - 1].i1 == i0) {
            a[n - 1].i1 = static_cast<int32_t>(i1);
            return;
        }
        Item& r = a[n++];
        r.kind = kRaw;
        r.i0 = static_cast<int32_t>(i0);
        r.i1 = static_cast<int32_t>(i1);
        r.tau = tau;
        r.E = 0;
    }
};

// turn item r (a piece) into a raw range reaching i1; its fields hold no terms
SS_HD void make_raw(Item& r, int64_t i1) {
    r.kind = kRaw;
    r.E = 0;
    r.i1 = static_cast<int32_t>(i1);
}

// Run elements [i0, i1): absorbed into the open piece (the output's last item, if it
// is a piece ending at i0), otherwise raw, reopening pieces at the simulated states.
// `state` is the simulated state before i0 when no piece is open; src(i) gives the
// terms (the accessor, or RawSrc over a raw item's inline terms).
// Requires o.n < o.cap on entry (or the last item open); keeps o.n <= o.cap.  When a
// raw element finds no free slot, the open piece it ends and the rest of the range
// become one raw item (re-simulated by a later merge or summed in the final pass).
template <class TermAt>
struct RawSrc {  // the terms of a raw item: inline first, then the accessor
    Item r;
    const TermAt* term;
    SS_HD double operator()(int64_t i) const { return raw_term(r, i, *term); }
};

template <class Src>
SS_HD void run_range(Out& o, double state, int64_t i0, int64_t i1, double tau, const Src& src) {
    bool open = o.n > 0 && o.last().kind != kRaw && o.last().i1 == i0;
    Item cur;  // the open piece, in registers while it absorbs
    if (open) cur = o.last();
    for (int64_t i = i0; i < i1; ++i) {
        const double t = src(i);
        if (open) {
            if (absorb(cur, t)) continue;
            state = cur.end[0];
            if (cur.i1 == cur.i0)
                --o.n;  // an empty piece carries nothing
            else
                o.last() = cur;
            open = false;
        }
        const bool joins = o.n > 0 && o.last().kind == kRaw && o.last().i1 == i;
        if (!joins && o.n == o.cap) {
            // no slot: the last item (a piece ending at i) and the rest become raw
            Item& r = o.last();
            make_raw(r, i1);
            if (o.n > 1 && o.a[o.n - 2].kind == kRaw && o.a[o.n - 2].i1 == r.i0) {
                o.a[o.n - 2].i1 = static_cast<int32_t>(i1);
                --o.n;
            }
            return;
        }
        o.push_raw1(i, t, tau);
        state = state + t;  // the simulated chain continues through the raw element
        if (o.n < o.cap && open_piece(state, tau, i + 1, cur)) {
            o.a[o.n++] = cur;
            open = true;
        }
    }
    if (open) {
        if (cur.i1 == cur.i0)
            --o.n;
        else
            o.last() = cur;
    }
}

// Simulate one thread's elements into o (empty) from the approximate start rep;
// exact: rep is the true state (+0.0 before element 0).
template <class TermAt>
SS_HD void simulate(Out& o, double rep, bool exact, int64_t i0, int64_t i1, double tau, const TermAt& term) {
    Item p;
    if (exact) {
        open_exact(rep, tau, i0, p);
        o.a[o.n++] = p;
    } else if (o.n < o.cap && open_piece(rep, tau, i0, p)) {
        o.a[o.n++] = p;
    }
    run_range(o, rep, i0, i1, tau, term);
}

// Append list R (items r[0..nr)) after the output's items, merging across the seam.
// In place: r lies at o.a + cap_base with cap_base >= o.n; once input k is read the
// output may use slots up to cap_base + k.
template <class TermAt>
SS_HD void append_list(Out& o, const Item* r, int nr, const TermAt& term, int cap_base) {
    for (int k = 0; k < nr; ++k) {
        const Item it = r[k];
        o.cap = cap_base + k + 1;
        if (o.n == 0) {
            o.a[o.n++] = it;
            continue;
        }
        Item& last = o.last();
        if (it.kind != kRaw) {
            if (last.kind != kRaw && last.i1 == it.i0 && compose(last, it)) continue;
            o.a[o.n++] = it;
            continue;
        }
        // raw input: re-simulate it from the open piece, if any
        if (last.kind != kRaw && last.i1 == it.i0) {
            run_range(o, 0.0, it.i0, it.i1, it.tau, RawSrc<TermAt>{it, &term});
        } else if (last.kind == kRaw && last.i1 == it.i0) {
            // adjacent raw runs: keep the inline terms that stay contiguous
            if (last.E == last.i1 - last.i0)
                for (int k = 0; k < it.E && last.E < kInline; ++k) last.tv[last.E++] = raw_term(it, it.i0 + k, term);
            last.i1 = it.i1;
        } else {
            o.a[o.n++] = it;
        }
    }
}

// Merge list R (lenR items at R) into list L (lenL items at L), R at or beyond L + lenL
// (any byte offset); returns the merged length (items at L).  The output grows into the
// gap and into R's slots as they are consumed.
template <class TermAt>
SS_HD int merge_ptr(Item* L, int lenL, Item* R, int lenR, const TermAt& term) {
    if (lenR == 0) return lenL;
    if (lenL == 1 && lenR == 1) {  // the common case: two single pieces, in registers
        Item a = *L;
        const Item b = *R;
        if (a.kind != kRaw && b.kind != kRaw && a.i1 == b.i0 && compose(a, b)) {
            *L = a;
            return 1;
        }
    }
    const int cap_base =
        static_cast<int>((reinterpret_cast<const char*>(R) - reinterpret_cast<const char*>(L)) / sizeof(Item));
    Out o{L, lenL, cap_base};
    append_list(o, R, lenR, term, cap_base);
    return o.n;
}

template <class TermAt>
SS_HD int merge_pair(Item* pool, int offL, int lenL, int offR, int lenR, const TermAt& term) {
    return merge_ptr(pool + offL, lenL, pool + offR, lenR, term);
}

// Keep at most cap items by turning the pieces with the fewest elements (next to a raw
// item, so the list shrinks) into raw ranges: their elements are re-simulated by a
// later merge or summed in the final pass.  The exact chain is kept.
SS_HD int truncate(Item* a, int n, int cap) {
    while (n > cap) {
        int best = -1;
        int64_t bl = INT64_MAX;
        for (int k = 0; k < n; ++k) {
            if (a[k].kind != kPiece) continue;
            const bool lraw = k > 0 && a[k - 1].kind == kRaw;
            const bool rraw = k + 1 < n && a[k + 1].kind == kRaw;
            if (!lraw && !rraw) continue;
            if (a[k].i1 - a[k].i0 < bl) {
                bl = a[k].i1 - a[k].i0;
                best = k;
            }
        }
        if (best < 0) {  // no such piece: the tail becomes one raw item
            Item& r = a[cap - 1];
            if (r.kind != kRaw) r.E = 0;
            r.kind = kRaw;
            r.i1 = a[n - 1].i1;
            return cap;
        }
        make_raw(a[best], a[best].i1);
        int lo = best, hi = best;  // the raw run around it
        if (lo > 0 && a[lo - 1].kind == kRaw) --lo;
        if (hi + 1 < n && a[hi + 1].kind == kRaw) ++hi;
        a[lo].i1 = a[hi].i1;  // a[lo]'s inline terms still describe its first elements
        const int gone = hi - lo;
        for (int k = lo + 1; k + gone < n; ++k) a[k] = a[k + gone];
        n -= gone;
    }
    return n;
}

// Apply a list to the true state s (the reference's running sum before r[0].i0).
template <class TermAt>
SS_HD double apply(const Item* r, int nr, double s, const TermAt& term, int64_t* fallback_elems) {
    for (int k = 0; k < nr; ++k) {
        const Item& it = r[k];
        if (it.kind == kExact && bits(s) == bits(it.rep[0])) {
            s = it.end[0];
            continue;
        }
        if (it.kind == kPiece) {
            const double d0 = s - it.rep[0];  // exact when |d0| < W (same binade as rep)
            if (std::fabs(d0) < it.W) {
                const int q = parity_units(d0, it.E);
                s = q ? it.end[1] + (s - it.rep[1]) : it.end[0] + d0;
                continue;
            }
        }
        // element by element, the terms read eight ahead of the chain: here they come from
        // global memory, and one dependent load per add made long fallbacks latency-bound
        // (C3's restarted FGMRES: ~40,000 such terms took 20 ms per sum)
        if (it.kind != kRaw && fallback_elems) *fallback_elems += it.i1 - it.i0;
        for (int64_t i = it.i0; i < it.i1; i += 8) {
            double tb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                tb[u] = i + u < it.i1 ? (it.kind != kRaw ? term(i + u) : raw_term(it, i + u, term)) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (i + u < it.i1) s = s + tb[u];
        }
    }
    return s;
}

}  // namespace ss
}  // namespace amgcu
