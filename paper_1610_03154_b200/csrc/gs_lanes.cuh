// Gauss-Seidel, lane per segment (relaxation.hpp:115-127; included by relax.cu).
//
// The forward sweep over a stencil level is a set of long chains (segments: maximal
// runs of rows each depending on its predecessor -- grid rows).  Here one LANE owns
// one segment and walks it row by row, every sweep in turn (segment-major).  A CTA
// serves 32 consecutive segments with one solver warp: in every warp iteration each
// lane relaxes its next row if the values it needs are there, so 32 rows advance per
// iteration and a segment trails its predecessor by about two iterations (its row x
// needs row x + 1 above).
//
// Roles (warps of one CTA):
//   solver (warp 0): lane l relaxes segment 32 * cta + l.  A row is its record's
//     prefix acc0 minus up to T terms in CSR order.  Every term is (a, source): the
//     source is a 16-byte (value, tag) cell in shared memory and the term is ready
//     when the tag equals the record's expected tag and the value is not the pending
//     sentinel.  Cells: a lane's ring of its last kLnRing published rows (tag =
//     sweep * n + row; this also serves x_{i-1}), a poll slot of the row record
//     (tag preset, value filled in by the poller), or a constant 1.0 cell for
//     products folded by the prefetcher (a * 1.0 == a exactly).  So a term costs three
//     shared loads, two compares and one multiply, with no branch; the lane subtracts
//     its terms in order up to the first one that is not ready and resumes from there
//     in the next iteration.  Publication: own ring cell and the sweep's global buffer.
//   prefetchers (kLnPf warps): build the row records kLnRows rows ahead of each
//     lane: load the CSR row, fold the prefix of products whose values are already
//     published into acc0, classify the rest.
//   poller (last warp): fills poll slots (values of other CTAs, or values not yet
//     published when the record was built) by relaxed global loads.
// Every row sum runs in the reference's order (acc -= a * x, product rounded first, no
// FMA), so the result is bit-identical to the CPU sweep.  Values are published in
// per-sweep buffers pre-filled with kPending.  A CTA takes its block of 32 segments from
// a ticket when it starts.  A row of sweep s reads rows earlier in (sweep, position)
// order: sweep s values of its own or earlier CTAs, and sweep s - 1 values of any CTA.
// Alone on the device every CTA is resident (the launcher keeps nctas <= SMs), so the
// earliest unfinished row always progresses.  On the second stream (candidate sweeps
// beside the aggregation, setup.cu) some CTAs may wait for SMs held by main-stream
// kernels; those kernels depend on nothing the sweeps hold (the main stream joins the
// sweeps only through an event, which holds no SM), so they finish, the SMs free up,
// every CTA becomes resident, and the same argument applies.

constexpr int kLnLanes = 32;  // segments per CTA
constexpr int kLnRb = 8;      // rows per record block
constexpr int kLnPf = 8;      // prefetch warps (each serves 4 lanes)
// Per-configuration sizes (template parameters): T terms per row record, BLK record
// blocks per lane (kLnRb * BLK rows of look-ahead), SLOTS poll slots per row, RING
// published rows kept per lane.  The launcher instantiates T = 8 (rows of up to 9
// entries: 3 blocks, 4 slots, 64-row rings) and T = 20 (up to 21 entries, e.g. the
// 19-point coarse operators: 2 blocks, 2 slots, 32-row rings), both ~210 KB.
constexpr int kLnThreads = (2 + kLnPf) * 32;

struct LnCell {
    unsigned long long v;  // value bits (kPending until known)
    int32_t tag;
    int32_t pad;
};

template <int T, int BLK, int SLOTS, int RING>
struct LnRec {
    static constexpr int kLnBlk = BLK;
    static constexpr int kLnRows = kLnRb * BLK;
    static constexpr int kLnSlots = SLOTS;
    static constexpr int kLnRing = RING;
    double ta[kLnRows][T][kLnLanes];              // a, or the folded product
    unsigned long long tw[kLnRows][T][kLnLanes];  // source cell smem address | expected tag << 32
    LnCell sv[kLnRows][kLnSlots][kLnLanes];       // poll slots
    uint32_t sa[kLnRows][kLnSlots][kLnLanes];     // poll slot: element offset in X
    double acc0[kLnRows][kLnLanes];
    double dinv[kLnRows][kLnLanes];
    int32_t meta[kLnRows][kLnLanes];  // nterm | nslot << 8 | slow << 16
    // rings: [0, 1] halo (the previous CTA's last two segments, streamed in by the
    // poller), [2 + l] lane l's published rows
    LnCell ring[kLnLanes + 2][kLnRing];
    LnCell one;  // (1.0, tag 0): source of folded products
    int32_t sq0[kLnLanes + 1];
    int32_t hq0[3];  // halo segments: [hq0[0], hq0[1]), [hq0[1], hq0[2] = sq0[0])
    int32_t ready[kLnLanes];     // record blocks prepared
    int32_t consumed[kLnLanes];  // rows finished
    int32_t live;                // the solver is running
};

template <int T, int BLK, int SLOTS, int RING>
constexpr size_t ln_smem_bytes() {
    return sizeof(LnRec<T, BLK, SLOTS, RING>);
}

// acquire / release on shared-memory flags.  In the shared state space the acquire
// load is a plain LDS (no fence: a generic-address atomic_ref would emit MEMBAR.SC,
// which waits for this thread's outstanding global stores -- microseconds for the
// solver, which publishes to global memory every row).
__device__ __forceinline__ int ld_acquire_cta(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
                 : "=r"(v)
                 : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p)))
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(int32_t* p, int32_t v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(p))),
                 "r"(v)
                 : "memory");
}
__device__ __forceinline__ void ld_cell(unsigned addr, unsigned long long& v, int32_t& tag) {
    unsigned lo, hi, t, p;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(lo), "=r"(hi), "=r"(t), "=r"(p)
                 : "r"(addr));
    v = (static_cast<unsigned long long>(hi) << 32) | lo;
    tag = static_cast<int32_t>(t);
}
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int T, int BLK, int SLOTS, int RING>
__global__ void __launch_bounds__(kLnThreads, 1)
    k_gs_lanes(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const double* __restrict__ va, const double* __restrict__ inv_diag, const double* __restrict__ b,
               int nsw, const int32_t* __restrict__ segs, int32_t nseg, double* __restrict__ X,
               unsigned int* __restrict__ ticket, unsigned long long* __restrict__ stats, unsigned poll_ns,
               unsigned pf_ns, int32_t ncol, size_t xcol_stride) {
    extern __shared__ unsigned long long ln_smem[];
    using Rec = LnRec<T, BLK, SLOTS, RING>;
    Rec& R = *reinterpret_cast<Rec*>(ln_smem);
    constexpr int kLnBlk = Rec::kLnBlk;
    constexpr int kLnRows = Rec::kLnRows;
    constexpr int kLnSlots = Rec::kLnSlots;
    constexpr int kLnRing = Rec::kLnRing;
    // prefetch: a row's entries (and then their published values) loaded in batches of
    constexpr int kPfChunk = 8;
    __shared__ unsigned int blk, colv;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // tickets interleave the columns (independent sweeps of the same matrix): ticket t is
    // block t / ncol of column t % ncol, so a block's predecessor in its column always
    // holds a smaller ticket
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        blk = t / static_cast<unsigned>(ncol);
        colv = t % static_cast<unsigned>(ncol);
    }
    __syncthreads();
    X += static_cast<size_t>(colv) * xcol_stride;
    if (b) b += static_cast<size_t>(colv) * static_cast<size_t>(n);
    const int32_t g0 = static_cast<int32_t>(blk) * kLnLanes;
    for (int e = threadIdx.x; e < (kLnLanes + 2) * kLnRing; e += blockDim.x) {
        R.ring[e / kLnRing][e % kLnRing].v = kPending;
        R.ring[e / kLnRing][e % kLnRing].tag = -1;
    }
    if (threadIdx.x <= kLnLanes) R.sq0[threadIdx.x] = segs[min(g0 + static_cast<int32_t>(threadIdx.x), nseg)];
    if (threadIdx.x < 3) R.hq0[threadIdx.x] = segs[max(g0 - 2 + static_cast<int32_t>(threadIdx.x), 0)];
    if (threadIdx.x < kLnLanes) {
        R.ready[threadIdx.x] = 0;
        R.consumed[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
        R.live = 1;
        R.one.v = static_cast<unsigned long long>(__double_as_longlong(1.0));
        R.one.tag = 0;
    }
    __syncthreads();
    const size_t stride = static_cast<size_t>(n);
    const int32_t qc0 = R.sq0[0];  // first row of this CTA's segments
    const int32_t hq0 = R.hq0[0];  // first row served by a ring (halo included)

    if (warp == 0) {
        // ---------------- solver ----------------
        const int32_t q0 = R.sq0[lane], len = R.sq0[lane + 1] - q0;
        const int32_t total = len * nsw;
        int32_t u = 0, kres = 0;
        int32_t s = 0, q = q0;  // sweep and row of row u
        int slot = 0;           // u % kLnRows
        double acc = 0.0;
        int32_t rdy = 0;  // record rows known to be prepared (acquired)
        // the current row's record in registers (loaded one iteration ahead when possible,
        // so the record round trip is off the critical path)
        bool have = false;
        int32_t meta = 0;
        double dq = 0.0;
        double ta[T];
        unsigned long long tw[T];
        long long ck[4] = {0, 0, 0, 0};
        if (stats && lane == 0) atomicMin(stats + 24, globaltimer_ns());
        long long iters = 0;
        while (true) {
            ++iters;
            const long long c0 = stats ? clock64() : 0;
            const bool act = u < total;
            if (!__any_sync(0xffffffffu, act)) break;
            bool fin = false;
            double xnew = 0.0;
            if (act) {
                if (!have) {
                    if (rdy <= u) rdy = ld_acquire_cta(&R.ready[lane]) * kLnRb;
                    if (rdy > u) {
                        meta = R.meta[slot][lane];
                        acc = R.acc0[slot][lane];
                        dq = R.dinv[slot][lane];
#pragma unroll
                        for (int k = 0; k < T; ++k) {
                            ta[k] = R.ta[slot][k][lane];
                            tw[k] = R.tw[slot][k][lane];
                        }
                        kres = 0;
                        have = true;
                    }
                }
                if (have) {
                    const int nt = meta & 0xff;
                    if (!(meta >> 16)) {
                        // chunks of 8 terms (register pressure for wide rows): resolve the
                        // chunk's cells, subtract in term order up to the first value that is
                        // not there yet
                        const unsigned live_m = ((1u << nt) - 1u) & ~((1u << kres) - 1u);
                        bool stopped = false;
                        int kstop = nt;
#pragma unroll
                        for (int cb = 0; cb < T; cb += 8) {
                            if (!stopped && cb < nt) {
                                unsigned long long vv[8];
                                int32_t tg[8];
#pragma unroll
                                for (int w = 0; w < 8; ++w)
                                    if (cb + w < T) ld_cell(static_cast<unsigned>(tw[cb + w]), vv[w], tg[w]);
                                double pk[8];
                                unsigned okc = 0u, evc = 0u;
#pragma unroll
                                for (int w = 0; w < 8; ++w) {
                                    if (cb + w < T) {
                                        const int32_t want = static_cast<int32_t>(tw[cb + w] >> 32);
                                        okc |= ((tg[w] == want && vv[w] != kPending) ? 1u : 0u) << w;
                                        evc |= (tg[w] > want ? 1u : 0u) << w;
                                        pk[w] = ta[cb + w] * __longlong_as_double(static_cast<long long>(vv[w]));
                                    }
                                }
                                const unsigned livec = (live_m >> cb) & 0xffu;
                                if (evc & livec) {
                                    // a ring value was overwritten before this lane read it (it
                                    // was published long ago; rare): read it from the sweep buffer
#pragma unroll
                                    for (int w = 0; w < 8; ++w) {
                                        if (cb + w < T && ((evc >> w) & 1u)) {
                                            const int32_t want = static_cast<int32_t>(tw[cb + w] >> 32);
                                            const unsigned long long bits =
                                                load_relaxed_bits(X + stride + static_cast<size_t>(want));
                                            if (bits != kPending) {
                                                okc |= 1u << w;
                                                pk[w] = ta[cb + w] * __longlong_as_double(static_cast<long long>(bits));
                                            }
                                        }
                                    }
                                }
                                const unsigned badc = ~okc & livec;
                                const int ks = badc ? cb + __ffs(badc) - 1 : min(nt, cb + 8);
#pragma unroll
                                for (int w = 0; w < 8; ++w) {
                                    // predicated, not branched: the subtraction chain is the
                                    // iteration's critical path
                                    const double d = acc - pk[w];
                                    acc = (cb + w < T && cb + w >= kres && cb + w < ks) ? d : acc;
                                }
                                if (badc) {
                                    stopped = true;
                                    kstop = ks;
                                }
                            }
                        }
                        kres = kstop;
                        fin = !stopped;
                    } else {
                        // slow row (more terms or pending values than the record holds): the
                        // CSR row from global memory, resumable at entry kres
                        const int32_t lo = rp[q], hi = rp[q + 1];
                        const double* xin = X + static_cast<size_t>(s) * stride;
                        const double* xo = X + static_cast<size_t>(s + 1) * stride;
                        bool stop = false;
                        for (int32_t e = lo + kres; e < hi && !stop; ++e) {
                            const int32_t j = ci[e];
                            if (j == q) {
                                ++kres;
                                continue;
                            }
                            const unsigned long long bits = load_relaxed_bits(j < q ? xo + j : xin + j);
                            if (bits == kPending) {
                                stop = true;
                            } else {
                                acc -= va[e] * __longlong_as_double(static_cast<long long>(bits));
                                ++kres;
                            }
                        }
                        fin = !stop;
                    }
                    if (fin) xnew = acc * dq;
                }
            }
            const long long c1 = stats ? clock64() : 0;
            if (stats) {
                const unsigned mfin = __ballot_sync(0xffffffffu, fin);
                const unsigned mact = __ballot_sync(0xffffffffu, act);
                const unsigned mrec = __ballot_sync(0xffffffffu, act && !have);
                if (lane == 0) {
                    atomicAdd(stats + 0, 1ull);
                    atomicAdd(stats + 1, static_cast<unsigned long long>(__popc(mfin)));
                    atomicAdd(stats + 2, static_cast<unsigned long long>(__popc(mact)));
                    atomicAdd(stats + 3, static_cast<unsigned long long>(__popc(mrec)));
                }
            }
            __syncwarp();  // every lane has read its cells before any ring cell is rewritten
            const long long c2 = stats ? clock64() : 0;
            if (fin) {
                const unsigned long long xb = static_cast<unsigned long long>(__double_as_longlong(xnew));
                // value and tag in one 16-byte store: a sibling lane's 16-byte read of the
                // cell never sees one without the other
                const unsigned ca = smem_addr(&R.ring[lane + 2][q & (kLnRing - 1)]);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ca), "r"(static_cast<unsigned>(xb)),
                             "r"(static_cast<unsigned>(xb >> 32)), "r"(static_cast<unsigned>(s * n + q)), "r"(0u)
                             : "memory");
                cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> out(
                    *reinterpret_cast<unsigned long long*>(X + static_cast<size_t>(s + 1) * stride + q));
                out.store(xb, cuda::memory_order_relaxed);
                ++u;
                if (++slot == kLnRows) slot = 0;
                if (++q == q0 + len) {
                    q = q0;
                    ++s;
                }
                vstore(&R.consumed[lane], u);
                // the next row's record, if prepared: its loads overlap the barrier and the
                // loop head
                have = false;
                if (u < total) {
                    if (rdy <= u) rdy = ld_acquire_cta(&R.ready[lane]) * kLnRb;
                    if (rdy > u) {
                        meta = R.meta[slot][lane];
                        acc = R.acc0[slot][lane];
                        dq = R.dinv[slot][lane];
#pragma unroll
                        for (int k = 0; k < T; ++k) {
                            ta[k] = R.ta[slot][k][lane];
                            tw[k] = R.tw[slot][k][lane];
                        }
                        kres = 0;
                        have = true;
                    }
                }
            }
            __syncwarp();  // lanes stay in step (skew between sibling segments is in iterations)
            if (stats) {
                const long long c3 = clock64();
                ck[0] += c1 - c0;
                ck[1] += c2 - c1;
                ck[2] += c3 - c2;
                ck[3] += c3 - c0;
            }
        }
        if (stats && lane == 0) {
            for (int e = 0; e < 4; ++e) atomicAdd(stats + 16 + e, static_cast<unsigned long long>(ck[e]));
            atomicMax(stats + 25, globaltimer_ns());
            atomicMax(stats + 26, static_cast<unsigned long long>(iters));
            atomicMax(stats + 27, static_cast<unsigned long long>(ck[3]));
        }
        if (lane == 0) vstore(&R.live, 0);
        return;
    }

    if (warp <= kLnPf) {
        // ---------------- prefetchers ----------------
        const int pw = warp - 1;
        const int l = pw * (kLnLanes / kLnPf) + lane / kLnRb;  // lane served by this thread
        const int r = lane % kLnRb;                            // row of the block
        const int32_t q0 = R.sq0[l], len = R.sq0[l + 1] - q0;
        const int32_t total = len * nsw;
        const int32_t nblocks = (total + kLnRb - 1) / kLnRb;
        const unsigned one_addr = smem_addr(&R.one);
        // Each pass serves, together, the lanes whose next block has a free slot (the
        // slot's previous block consumed); a lane never waits on another lane's
        // consumption (it may need values of a row that lane reaches only with new records).
        int32_t bi = 0;  // next block of this thread's lane
        while (__any_sync(0xffffffffu, bi < nblocks)) {
            const bool go = bi < nblocks && (bi < kLnBlk || ld_acquire_cta(&R.consumed[l]) >= (bi - kLnBlk + 1) * kLnRb);
            if (!__any_sync(0xffffffffu, go)) {
                __nanosleep(pf_ns);
                continue;
            }
            const int32_t u = bi * kLnRb + r;
            const int slot = u % kLnRows;
            if (go && u < total) {
                const int32_t s = u / len;
                const int32_t q = q0 + (u - s * len);
                const double* xin = X + static_cast<size_t>(s) * stride;
                const double* xo = X + static_cast<size_t>(s + 1) * stride;
                const int32_t lo = rp[q], hi = rp[q + 1];
                double acc = b ? b[q] : 0.0;
                const double dq = inv_diag[q];
                int nt = 0, nslot = 0;
                bool slow = false, prefix = true;
                for (int32_t e0 = lo; e0 < hi; e0 += kPfChunk) {
                    int32_t jj[kPfChunk];
                    double aa[kPfChunk];
                    unsigned long long xv[kPfChunk];
#pragma unroll
                    for (int w = 0; w < kPfChunk; ++w) {
                        jj[w] = q;
                        aa[w] = 0.0;
                        if (e0 + w < hi) {
                            jj[w] = ci[e0 + w];
                            aa[w] = va[e0 + w];
                        }
                    }
                    // values that are published now: every old value (previous sweep; sweep 0
                    // reads the input x) and new values of rows outside this CTA's segments
#pragma unroll
                    for (int w = 0; w < kPfChunk; ++w) {
                        const int32_t j = jj[w];
                        xv[w] = kPending;
                        if (j > q)
                            xv[w] = s == 0 ? static_cast<unsigned long long>(__double_as_longlong(__ldcg(xin + j)))
                                           : load_relaxed_bits(xin + j);
                        else if (j < hq0)
                            xv[w] = load_relaxed_bits(xo + j);
                    }
#pragma unroll
                    for (int w = 0; w < kPfChunk; ++w) {
                        const int32_t j = jj[w];
                        if (j == q) continue;  // diagonal or padding
                        if (xv[w] != kPending) {
                            const double p = aa[w] * __longlong_as_double(static_cast<long long>(xv[w]));
                            if (prefix) {
                                acc -= p;
                                continue;
                            }
                            if (nt >= T) {
                                slow = true;
                                continue;
                            }
                            R.ta[slot][nt][l] = p;
                            R.tw[slot][nt][l] = one_addr;  // (1.0, tag 0)
                            ++nt;
                            continue;
                        }
                        prefix = false;
                        unsigned addr;
                        int32_t want;
                        if (j < q && j >= hq0) {
                            // earlier row of a segment of this CTA (own included) or of the
                            // previous CTA's last two: its ring cell
                            int rg;
                            if (j >= qc0) {
                                // the producing lane: walk back from the own one (stencil
                                // couplings reach a segment or two)
                                int l2 = l;
                                while (R.sq0[l2] > j) --l2;
                                rg = l2 + 2;
                            } else {
                                rg = j >= R.hq0[1] ? 1 : 0;
                            }
                            addr = smem_addr(&R.ring[rg][j & (kLnRing - 1)]);
                            want = s * n + j;
                        } else {
                            if (nslot >= kLnSlots) {
                                slow = true;
                                continue;
                            }
                            R.sv[slot][nslot][l].v = kPending;
                            R.sv[slot][nslot][l].tag = 0;
                            R.sa[slot][nslot][l] =
                                static_cast<uint32_t>(static_cast<size_t>(j > q ? s : s + 1) * stride + j);
                            addr = smem_addr(&R.sv[slot][nslot][l]);
                            want = 0;
                            ++nslot;
                        }
                        if (nt >= T) {
                            slow = true;
                            continue;
                        }
                        R.ta[slot][nt][l] = aa[w];
                        R.tw[slot][nt][l] = addr | (static_cast<unsigned long long>(static_cast<uint32_t>(want)) << 32);
                        ++nt;
                    }
                }
                // unused term cells: the constant cell (never subtracted: k >= nt)
                for (int k = nt; k < T; ++k) R.tw[slot][k][l] = one_addr;
                R.acc0[slot][l] = slow ? (b ? b[q] : 0.0) : acc;
                R.dinv[slot][l] = dq;
                R.meta[slot][l] = slow ? (1 << 16) : (nt | (nslot << 8));
            }
            __syncwarp();
            if (go) {
                if (r == 0) st_release_cta(&R.ready[l], bi + 1);
                ++bi;
            }
        }
        return;
    }

    // ---------------- poller ----------------
    // A pass finds the solver lanes whose next kLnRb rows hold a pending poll slot (thread
    // = solver lane); each such lane's (row, slot) pairs are then loaded by the whole warp
    // at once (thread = row * 4 + slot), so one global round trip serves a lane's window.
    // It also streams the halo: lanes 0-15 / 16-31 follow the previous CTA's last two
    // segments in (sweep, row) order, 16 rows per round trip, and copy every published
    // value, in order, into the halo ring with one 16-byte store (value and tag together).
    {
        const int32_t total_l = (R.sq0[lane + 1] - R.sq0[lane]) * nsw;
        const int hh = lane >> 4;
        const int32_t hbase = R.hq0[hh], hlen = R.hq0[hh + 1] - hbase;
        const int32_t htotal = hlen * nsw;
        int32_t hcur = 0;  // halo rows copied so far (uniform within a 16-lane group)
        unsigned ns = 0;
        while (__shfl_sync(0xffffffffu, vload(&R.live), 0)) {
            bool hprog = false;
            {
                const int32_t hu = hcur + (lane & 15);
                bool ok = false;
                unsigned long long bits = kPending;
                int32_t hs = 0, hq = 0;
                if (hu < htotal) {
                    hs = hu / hlen;
                    hq = hbase + (hu - hs * hlen);
                    bits = load_relaxed_bits(X + static_cast<size_t>(hs + 1) * stride + hq);
                    ok = bits != kPending;
                }
                const unsigned okm = __ballot_sync(0xffffffffu, ok);
                const unsigned gm = (okm >> (hh * 16)) & 0xffffu;
                const int pre = __ffs(~gm) - 1;  // ready rows from the group's cursor on
                if ((lane & 15) < pre) {
                    const unsigned a = smem_addr(&R.ring[hh][hq & (kLnRing - 1)]);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                                 "r"(static_cast<unsigned>(bits)), "r"(static_cast<unsigned>(bits >> 32)),
                                 "r"(static_cast<unsigned>(hs * n + hq)), "r"(0u)
                                 : "memory");
                }
                hcur += pre;
                hprog = pre > 0;
            }
            const int32_t u0 = vload(&R.consumed[lane]);
            const int32_t uready = min(ld_acquire_cta(&R.ready[lane]) * kLnRb, total_l);
            bool pend = false;
            for (int32_t u = u0; u < min(u0 + kLnRb, uready) && !pend; ++u) {
                const int slot = u % kLnRows;
                const int32_t meta = R.meta[slot][lane];
                if (meta >> 16) continue;
                const int nsl = (meta >> 8) & 0xff;
                for (int k = 0; k < nsl; ++k) pend = pend || vload(&R.sv[slot][k][lane].v) == kPending;
            }
            unsigned mask = __ballot_sync(0xffffffffu, pend);
            const bool any = mask != 0u;
            bool progress = false;
            while (mask) {
                const int L = __ffs(mask) - 1;
                mask &= mask - 1;
                const int32_t u0L = __shfl_sync(0xffffffffu, u0, L);
                const int32_t urL = __shfl_sync(0xffffffffu, uready, L);
                const int32_t u = u0L + lane / kLnSlots;
                const int k = lane % kLnSlots;
                if (u < min(u0L + kLnRb, urL)) {
                    const int slot = u % kLnRows;
                    const int32_t meta = R.meta[slot][L];
                    if (!(meta >> 16) && k < ((meta >> 8) & 0xff) && vload(&R.sv[slot][k][L].v) == kPending) {
                        const unsigned long long bits = load_relaxed_bits(X + R.sa[slot][k][L]);
                        if (bits != kPending) {
                            vstore(&R.sv[slot][k][L].v, bits);
                            progress = true;
                        }
                    }
                }
            }
            // back off between passes (the shared-memory pipe is the solver's critical path)
            if (__any_sync(0xffffffffu, progress || hprog) || any) {
                ns = poll_ns;
            } else {
                ns = ns ? min(2 * ns, 1024u) : poll_ns;
            }
            if (ns) __nanosleep(ns);
        }
    }
}
