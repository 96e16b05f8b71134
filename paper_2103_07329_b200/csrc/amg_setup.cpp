// amg_setup.cpp -- native host restatement of the reference AMG setup and of
// the Chebyshev eigenvalue-bound estimate.  Output is bitwise identical to
// the reference (pinned by tests/test_setup_native.py against
// tests/golden/hierarchies.npz), so the hierarchy uploaded to the GPU is the
// reference's hierarchy -- produced ~100x faster than its Python loops.
//
//   strength_graph   src/amg.py:55-78    classical negative-coupling rule
//   coarsen          src/amg.py:89-124   index-ordered greedy C/F split
//   interpolate      src/amg.py:127-182  direct interpolation (numpy pairwise
//                                        sums reproduced exactly)
//   galerkin         src/amg.py:185-196  (R @ A) @ P with scipy's SMMP order:
//                                        unsorted intermediate rows, exact-zero
//                                        drop, then sort
//   setup            src/amg.py:254-308  level loop, stall cut, retry once,
//                                        mixed precision (levels >= 1 float32)
//   estimate_eig_bounds  src/solvers.py:486-517
//
// Compiled with -ffp-contract=off and no -march flags: every multiply-add is
// separately rounded, like the x86-64 baseline builds of numpy/scipy.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "../../include/mrsolve_b200.h"
#include "spgemm.h"

namespace {

struct Csr {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> rp;
    std::vector<int64_t> ci;
    std::vector<double> v;
    int64_t nnz() const { return (int64_t)ci.size(); }
};

constexpr int8_t U = 0, C = 1, F = 2;

// Row-parallel phases (strength, Galerkin products, row sorts) run on host
// threads: every output row is computed by one thread with the same
// per-row operation order as the sequential code, so the hierarchy is
// bitwise the same for any thread count.  MRS_SETUP_THREADS overrides.
int setup_threads() {
    static int t = 0;
    if (!t) {
        const char* e = getenv("MRS_SETUP_THREADS");
        t = e ? atoi(e) : (int)std::thread::hardware_concurrency();
        t = std::max(1, std::min(t, 16));
    }
    return t;
}

// fn(lo, hi, part) over `parts` contiguous row ranges of [0, n).
template <class Fn> void for_row_parts(int64_t n, int parts, Fn fn) {
    if (parts <= 1 || n < 4096) { fn(0, n, 0); return; }
    std::vector<std::thread> th;
    for (int p = 0; p < parts; ++p) {
        const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
        th.emplace_back([=, &fn] { fn(lo, hi, p); });
    }
    for (auto& t : th) t.join();
}

// Rows built per part (count, columns, values), concatenated in row order.
struct RowParts {
    std::vector<std::vector<int64_t>> len, ci;
    std::vector<std::vector<double>> v;
    explicit RowParts(int parts) : len(parts), ci(parts), v(parts) {}
    void into(Csr& out) {
        out.rp.assign(out.nrows + 1, 0);
        int64_t row = 0, total = 0;
        for (size_t p = 0; p < len.size(); ++p)
            for (int64_t l : len[p]) { total += l; out.rp[++row] = total; }
        out.ci.clear(); out.v.clear();
        out.ci.reserve(total); out.v.reserve(total);
        for (size_t p = 0; p < len.size(); ++p) {
            out.ci.insert(out.ci.end(), ci[p].begin(), ci[p].end());
            out.v.insert(out.v.end(), v[p].begin(), v[p].end());
            std::vector<int64_t>().swap(ci[p]);
            std::vector<double>().swap(v[p]);
        }
    }
};

// numpy's pairwise summation (loops_utils.h, PW_BLOCKSIZE 128) for a
// contiguous float64 array: what `arr.sum()` computes.
double pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

// Transpose with sorted output columns (scipy csr -> csc -> csr).
Csr transpose(const Csr& A) {
    Csr T;
    T.nrows = A.ncols; T.ncols = A.nrows;
    T.rp.assign(T.nrows + 1, 0);
    for (int64_t k = 0; k < A.nnz(); ++k) T.rp[A.ci[k] + 1]++;
    for (int64_t i = 0; i < T.nrows; ++i) T.rp[i + 1] += T.rp[i];
    T.ci.resize(A.nnz()); T.v.resize(A.nnz());
    std::vector<int64_t> pos(T.rp.begin(), T.rp.end() - 1);
    for (int64_t i = 0; i < A.nrows; ++i)
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            int64_t p = pos[A.ci[k]]++;
            T.ci[p] = i; T.v[p] = A.v[k];
        }
    return T;
}

// scipy csr_matmat (sparsetools/csr.h): per output row a linked list of
// touched columns (head insertion), sums accumulated in traversal order,
// exact zeros dropped, row emitted in list order (NOT sorted).
Csr matmat(const Csr& A, const Csr& B) {
    Csr Cm;
    Cm.nrows = A.nrows; Cm.ncols = B.ncols;
    // dense per-thread scratch of B.ncols entries: cap the threads by memory
    const int parts = std::max<int>(1, std::min<int64_t>(setup_threads(),
                                                         (int64_t)(2e9 / (16.0 * (B.ncols + 1)))));
    RowParts rows(parts);
    for_row_parts(A.nrows, parts, [&](int64_t r0, int64_t r1, int part) {
        std::vector<int64_t> next(B.ncols, -1);
        std::vector<double> sums(B.ncols, 0.0);
        auto& len = rows.len[part];
        auto& oc = rows.ci[part];
        auto& ov = rows.v[part];
        for (int64_t i = r0; i < r1; ++i) {
            int64_t head = -2, length = 0, kept = 0;
            for (int64_t jj = A.rp[i]; jj < A.rp[i + 1]; ++jj) {
                const int64_t j = A.ci[jj];
                const double v = A.v[jj];
                for (int64_t kk = B.rp[j]; kk < B.rp[j + 1]; ++kk) {
                    const int64_t k = B.ci[kk];
                    sums[k] += v * B.v[kk];
                    if (next[k] == -1) { next[k] = head; head = k; ++length; }
                }
            }
            for (int64_t jj = 0; jj < length; ++jj) {
                if (sums[head] != 0) { oc.push_back(head); ov.push_back(sums[head]); ++kept; }
                int64_t tmp = head;
                head = next[head];
                next[tmp] = -1;
                sums[tmp] = 0;
            }
            len.push_back(kept);
        }
    });
    rows.into(Cm);
    return Cm;
}

void sort_rows(Csr& A) {
    for_row_parts(A.nrows, setup_threads(), [&](int64_t r0, int64_t r1, int) {
        std::vector<std::pair<int64_t, double>> row;
        for (int64_t i = r0; i < r1; ++i) {
            int64_t lo = A.rp[i], hi = A.rp[i + 1];
            bool sorted = true;
            for (int64_t k = lo + 1; k < hi && sorted; ++k) sorted = A.ci[k - 1] <= A.ci[k];
            if (sorted) continue;
            row.clear();
            for (int64_t k = lo; k < hi; ++k) row.emplace_back(A.ci[k], A.v[k]);
            std::sort(row.begin(), row.end(),
                      [](const auto& a, const auto& b) { return a.first < b.first; });
            for (int64_t k = lo; k < hi; ++k) { A.ci[k] = row[k - lo].first; A.v[k] = row[k - lo].second; }
        }
    });
}

// strength_graph (amg.py:55-78): S[i,j] iff j != i and
// -a_ij >= theta * max_k(-a_ik) with a positive row max.  Structure only.
Csr strength(const Csr& A, double theta) {
    Csr S;
    S.nrows = A.nrows; S.ncols = A.ncols;
    const int parts = setup_threads();
    RowParts rows(parts);
    for_row_parts(A.nrows, parts, [&](int64_t r0, int64_t r1, int part) {
        for (int64_t i = r0; i < r1; ++i) {
            double rowmax = 0.0;
            int64_t kept = 0;
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
                if (A.ci[k] != i) rowmax = std::max(rowmax, -A.v[k]);
            if (rowmax > 0) {
                const double thr = theta * rowmax;
                for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
                    if (A.ci[k] != i && -A.v[k] >= thr) {
                        rows.ci[part].push_back(A.ci[k]);
                        rows.v[part].push_back(1.0);
                        ++kept;
                    }
            }
            rows.len[part].push_back(kept);
        }
    });
    rows.into(S);
    return S;
}

// coarsen (amg.py:89-124)
std::vector<int8_t> split(const Csr& S, bool aggressive, int num_paths) {
    const int64_t n = S.nrows;
    Csr ST = transpose(S);
    std::vector<int8_t> st(n, U);
    std::vector<int32_t> cnt(aggressive ? n : 0, 0);
    std::vector<int64_t> touched;
    for (int64_t i = 0; i < n; ++i) {
        if (st[i] != U) continue;
        st[i] = C;
        const int64_t lo = ST.rp[i], hi = ST.rp[i + 1];
        for (int64_t k = lo; k < hi; ++k)
            if (st[ST.ci[k]] == U) st[ST.ci[k]] = F;
        if (aggressive && hi > lo) {
            touched.clear();
            for (int64_t k = lo; k < hi; ++k) {
                const int64_t q = ST.ci[k];
                for (int64_t kk = ST.rp[q]; kk < ST.rp[q + 1]; ++kk) {
                    const int64_t j = ST.ci[kk];
                    if (cnt[j]++ == 0) touched.push_back(j);
                }
            }
            for (int64_t j : touched) {
                if (cnt[j] >= num_paths && st[j] == U && j != i) st[j] = F;
            }
            for (int64_t j : touched) cnt[j] = 0;
        }
    }
    return st;
}

// interpolate (amg.py:127-182).  Returns false with the degenerate F rows.
bool interp(const Csr& A, const Csr& S, const std::vector<int8_t>& st, Csr& P,
            std::vector<int64_t>& bad) {
    const int64_t n = A.nrows;
    std::vector<int64_t> cmap(n, -1);
    int64_t nc = 0;
    for (int64_t i = 0; i < n; ++i)
        if (st[i] == C) cmap[i] = nc++;
    P = Csr();
    P.nrows = n; P.ncols = nc;
    bad.clear();
    // rows are independent: row-parallel on the host threads, each row computed
    // exactly as in the sequential loop (same pairwise sums, same entry order)
    const int parts = std::max<int>(1, std::min<int64_t>(setup_threads(),
                                                         (int64_t)(2e9 / (double)(n + 1))));
    RowParts rows(parts);
    std::vector<std::vector<int64_t>> badp(parts);
    for_row_parts(n, parts, [&](int64_t r0, int64_t r1, int part) {
        std::vector<double> diag, off, sel;
        std::vector<int64_t> selc;
        std::vector<char> strong_mark(n, 0);
        auto& len = rows.len[part];
        auto& oc = rows.ci[part];
        auto& ov = rows.v[part];
        for (int64_t i = r0; i < r1; ++i) {
            if (st[i] == C) {
                oc.push_back(cmap[i]); ov.push_back(1.0);
                len.push_back(1);
                continue;
            }
            for (int64_t k = S.rp[i]; k < S.rp[i + 1]; ++k) strong_mark[S.ci[k]] = 1;
            diag.clear(); off.clear(); sel.clear(); selc.clear();
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const int64_t c = A.ci[k];
                if (c == i) diag.push_back(A.v[k]);
                else off.push_back(A.v[k]);
                if (strong_mark[c] && st[c] == C) { sel.push_back(A.v[k]); selc.push_back(c); }
            }
            for (int64_t k = S.rp[i]; k < S.rp[i + 1]; ++k) strong_mark[S.ci[k]] = 0;
            if (sel.empty()) {
                badp[part].push_back(i);
                len.push_back(0);
                continue;
            }
            const double a_ii = pairwise_sum(diag.data(), (int64_t)diag.size());
            const double off_sum = pairwise_sum(off.data(), (int64_t)off.size());
            const double strong_sum = pairwise_sum(sel.data(), (int64_t)sel.size());
            const double ratio = off_sum / strong_sum;
            for (size_t q = 0; q < sel.size(); ++q) {
                oc.push_back(cmap[selc[q]]);
                ov.push_back((-(sel[q] / a_ii)) * ratio);
            }
            len.push_back((int64_t)sel.size());
        }
    });
    rows.into(P);
    for (auto& bp : badp) bad.insert(bad.end(), bp.begin(), bp.end());
    return bad.empty();
}

struct Level {
    Csr A, P, R;
    bool hasP = false;
    bool reduced = false;
    std::vector<float> Af, Pf, Rf;       // float32 copies on reduced levels
    std::vector<uint32_t> Aci, Pci, Rci; // 32-bit column copies for export
};

}  // namespace

struct mrs_hierarchy {
    std::vector<Level> levels;
};

namespace {

Csr from_host(const mrs_host_csr* h) {
    Csr A;
    A.nrows = h->nrows; A.ncols = h->ncols;
    A.rp.assign(h->row_ptr, h->row_ptr + h->nrows + 1);
    A.ci.resize(h->nnz); A.v.resize(h->nnz);
    for_row_parts(h->nnz, setup_threads(), [&](int64_t k0, int64_t k1, int) {
        for (int64_t k = k0; k < k1; ++k) {
            A.ci[k] = h->idx_bytes == 4 ? ((const uint32_t*)h->col_idx)[k]
                    : h->idx_bytes == 2 ? ((const uint16_t*)h->col_idx)[k]
                                        : ((const uint8_t*)h->col_idx)[k];
            A.v[k] = h->val_bytes == 8 ? ((const double*)h->values)[k]
                                       : (double)((const float*)h->values)[k];
        }
    });
    return A;
}

void export_csr(const Csr& A, bool reduced, std::vector<float>& vf, std::vector<uint32_t>& ci) {
    ci.resize(A.nnz());
    if (reduced) vf.resize(A.nnz());
    for_row_parts(A.nnz(), setup_threads(), [&](int64_t k0, int64_t k1, int) {
        for (int64_t k = k0; k < k1; ++k) ci[k] = (uint32_t)A.ci[k];
        if (reduced)
            for (int64_t k = k0; k < k1; ++k) vf[k] = (float)A.v[k];
    });
}

}  // namespace

extern "C" {

int mrs_amg_setup(const mrs_host_csr* Ah, const mrs_amg_params* prm, mrs_hierarchy** out) {
    if (!Ah || !prm || !out) return MRS_ERR_ARG;
    if (Ah->nrows != Ah->ncols) return MRS_ERR_ARG;
    if (!(prm->strength_threshold > 0.0 && prm->strength_threshold < 1.0)) return MRS_ERR_ARG;
    if (prm->coarse_matrix_size < 1 || prm->max_levels < 2 || prm->num_paths < 1) return MRS_ERR_ARG;
    std::vector<Csr> chain;
    chain.push_back(from_host(Ah));
    sort_rows(chain.back());
    std::vector<Csr> Ps, Rs;
    const bool timing = getenv("MRS_SETUP_TIMING") != nullptr;
    double tphase[6] = {0, 0, 0, 0, 0, 0};
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    while (chain.back().nrows > prm->coarse_matrix_size && (int)chain.size() < prm->max_levels) {
        const Csr& M = chain.back();
        auto t0 = now();
        Csr S = strength(M, prm->strength_threshold);
        auto t1 = now();
        const bool agg = (int)chain.size() - 1 < prm->agg_num_levels;
        std::vector<int8_t> st = split(S, agg, prm->num_paths);
        auto t2 = now();
        Csr P;
        std::vector<int64_t> bad;
        if (!interp(M, S, st, P, bad)) {
            for (int64_t r : bad) st[r] = C;
            if (!interp(M, S, st, P, bad)) return MRS_ERR_DEGENERATE;
        }
        auto t3 = now();
        const int64_t ncoarse = P.ncols;
        if (ncoarse == 0 || (double)ncoarse > prm->stall_ratio * (double)M.nrows) break;
        Csr R = transpose(P);
        Csr Ac;
        auto t4 = now(), t5 = t4;
        {
            // Galerkin product on the GPU when one is present (spgemm.cu: bitwise
            // the host products below), else on the host threads
            const mrs::HostCsrView vR{R.nrows, R.ncols, R.rp.data(), R.ci.data(), R.v.data()};
            const mrs::HostCsrView vA{M.nrows, M.ncols, M.rp.data(), M.ci.data(), M.v.data()};
            const mrs::HostCsrView vP{P.nrows, P.ncols, P.rp.data(), P.ci.data(), P.v.data()};
            Ac.nrows = R.nrows; Ac.ncols = P.ncols;
            if (mrs::galerkin_gpu(vR, vA, vP, Ac.rp, Ac.ci, Ac.v)) {
                t4 = t5 = now();
            } else {
                Csr RA = matmat(R, M);
                t4 = now();
                Ac = matmat(RA, P);
                t5 = now();
                sort_rows(Ac);
            }
        }
        auto t6 = now();
        tphase[0] += secs(t0, t1); tphase[1] += secs(t1, t2); tphase[2] += secs(t2, t3);
        tphase[3] += secs(t3, t4); tphase[4] += secs(t4, t5); tphase[5] += secs(t5, t6);
        Ps.push_back(std::move(P));
        Rs.push_back(std::move(R));
        chain.push_back(std::move(Ac));
    }
    if (timing)
        fprintf(stderr, "[mrs_amg_setup] strength %.2fs split %.2fs interp %.2fs RA %.2fs RAP %.2fs sort %.2fs (%d threads; %lld Galerkin products on the GPU so far: those count under RA)\n",
                tphase[0], tphase[1], tphase[2], tphase[3], tphase[4], tphase[5], setup_threads(),
                (long long)mrs::galerkin_gpu_count());
    mrs_hierarchy* h = new mrs_hierarchy();
    h->levels.resize(chain.size());
    for (size_t l = 0; l < chain.size(); ++l) {
        Level& lv = h->levels[l];
        lv.reduced = prm->mixed_precision && l > 0;
        lv.A = std::move(chain[l]);
        export_csr(lv.A, lv.reduced, lv.Af, lv.Aci);
        if (l < Ps.size()) {
            lv.hasP = true;
            lv.P = std::move(Ps[l]);
            lv.R = std::move(Rs[l]);
            export_csr(lv.P, lv.reduced, lv.Pf, lv.Pci);
            export_csr(lv.R, lv.reduced, lv.Rf, lv.Rci);
        }
    }
    *out = h;
    return MRS_OK;
}

int mrs_hier_nlevels(const mrs_hierarchy* h) { return h ? (int)h->levels.size() : 0; }

int mrs_hier_get(const mrs_hierarchy* h, int32_t level, int32_t which, mrs_host_csr* out) {
    if (!h || !out || level < 0 || level >= (int)h->levels.size()) return MRS_ERR_ARG;
    const Level& lv = h->levels[level];
    const Csr* M;
    const std::vector<float>* vf;
    const std::vector<uint32_t>* ci;
    switch (which) {
    case 0: M = &lv.A; vf = &lv.Af; ci = &lv.Aci; break;
    case 1: if (!lv.hasP) return MRS_ERR_ARG; M = &lv.P; vf = &lv.Pf; ci = &lv.Pci; break;
    case 2: if (!lv.hasP) return MRS_ERR_ARG; M = &lv.R; vf = &lv.Rf; ci = &lv.Rci; break;
    default: return MRS_ERR_ARG;
    }
    out->nrows = M->nrows; out->ncols = M->ncols; out->nnz = M->nnz();
    out->row_ptr = M->rp.data();
    out->col_idx = ci->data();
    out->idx_bytes = 4;
    if (lv.reduced) { out->values = vf->data(); out->val_bytes = 4; }
    else { out->values = M->v.data(); out->val_bytes = 8; }
    return MRS_OK;
}

void mrs_hier_destroy(mrs_hierarchy* h) { delete h; }

// estimate_eig_bounds (solvers.py:486-517): power iteration on D^-1 A with
// the caller's start vector (numpy default_rng(12345).standard_normal(n)).
int mrs_eig_bounds(const mrs_host_csr* Ah, int32_t iterations, uint64_t, const double* start,
                   double* lmin, double* lmax) {
    if (!Ah || !start || !lmin || !lmax) return MRS_ERR_ARG;
    Csr A = from_host(Ah);
    const int64_t n = A.nrows;
    std::vector<double> d(n, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        bool found = false;
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (A.ci[k] == i) { d[i] = A.v[k]; found = true; break; }
        if (!found || d[i] == 0.0) return MRS_ERR_SINGULAR;
    }
    std::vector<double> vec(start, start + n), w(n);
    double lam = 1.0;
    for (int it = 0; it < iterations; ++it) {
        for (int64_t i = 0; i < n; ++i) {       // csr_spmv ASSIGN, entry order
            double acc = 0.0;
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) acc += A.v[k] * vec[A.ci[k]];
            w[i] = acc;
        }
        for (int64_t i = 0; i < n; ++i) w[i] = w[i] / d[i];
        double num = 0.0, den = 0.0, ww = 0.0;   // dot_partial: sequential folds
        for (int64_t i = 0; i < n; ++i) num += vec[i] * w[i];
        for (int64_t i = 0; i < n; ++i) den += vec[i] * vec[i];
        lam = num / den;
        for (int64_t i = 0; i < n; ++i) ww += w[i] * w[i];
        const double wn = std::sqrt(ww);
        if (wn == 0.0) break;
        for (int64_t i = 0; i < n; ++i) vec[i] = w[i] / wn;
    }
    const double lm = 1.1 * std::fabs(lam);
    *lmin = lm / 30.0;
    *lmax = lm;
    return MRS_OK;
}

}  // extern "C"
