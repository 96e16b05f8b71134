// solver.cu -- the solver plan: uploaded hierarchy, static kernel schedule
// of one solve, and its CUDA-graph execution with a device-side while loop.
//
// Replaces solvers.prepare(...).run(B, X) (src/solvers.py:850-959) for
//   CG         (cg_solve, solvers.py:152-188)
//   BiCGStab   (_bicgstab_classical, solvers.py:219-293)
//   RBiCGStab  (_bicgstab_reordered, solvers.py:296-364)
//   PBiCGStab  (_bicgstab_pipelined, solvers.py:367-479)
// preconditioned by nothing, Jacobi sweeps (_SweepPrecond, :716-726) or a
// MultiGrid V-cycle (solvers.py:615-675) with Jacobi (blas2.py:165-185) or
// Chebyshev (solvers.py:520-571) smoothing and a dense coarsest solve.
//
// Execution model: the whole solve (prologue, iteration body, true-residual
// epilogue) is a static sequence of kernel launches whose scalar decisions
// (alpha, beta, omega, convergence, breakdown) are taken ON THE DEVICE by the
// reduction epilogues (reduce.cuh).  It is captured once into a CUDA graph
// whose iteration body sits under a conditional WHILE node that the
// epilogues drive with cudaGraphSetConditional: one graph launch per solve,
// no host round trip per iteration.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "comm.h"
#include "sgs.cuh"
#include "sgs_sched.h"
#include "dispatch.h"

using namespace mrs;

namespace {

using Launch = std::function<cudaError_t(cudaStream_t)>;

struct LevelDev {
    DevCsr A, P, R;          // P: n_l x n_{l+1}, R: n_{l+1} x n_l (local blocks when distributed)
    double* d = nullptr;     // diagonal (full precision of stored values)
    // multi-GPU layout; single GPU: nloc = rows, no halos
    int64_t nloc = 0;        // rows this rank owns (replicated level: all rows)
    int64_t vrows = 0;       // allocated rows of level vectors (own + largest halo; gather pad)
    bool replicated = false; // agglomerated: every rank holds the whole level
    bool f32 = false;        // this level's V-cycle vectors are float (plan vec32)
    int64_t slice_row0 = 0, slice_rows = 0;   // agglomeration: my restricted slice, allgather count
    Halo hA, hR, hP;         // operand exchanges of A_l x, R_l r, P_l x_{l+1}
    double lmin = 0, lmax = 0;
    double* b = nullptr;     // rhs buffer (levels >= 1)
    double* xa = nullptr;
    double* xb = nullptr;
    double* r = nullptr;
    double* dva = nullptr;
    double* dvb = nullptr;
    // Gauss-Seidel: level schedules of the forward [0] / backward [1] sweep
    int4* sgs_meta[2] = {nullptr, nullptr};   // (row, lo, hi, diag entry), schedule order
    int32_t* sgs_lptr[2] = {nullptr, nullptr};
    int sgs_nlev[2] = {0, 0};
    bool sgs = false;
};

// halo/compute overlap only where the interior run is worth a second launch
constexpr int64_t kMinOverlapRows = 2048;

template <typename T> T* dalloc(size_t n, std::vector<void*>& owned) {
    void* p = nullptr;
    if (n == 0) n = 1;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
    owned.push_back(p);
    return (T*)p;
}

}  // namespace

struct mrs_plan {
    mrs_plan_desc desc{};
    int64_t n = 0, m = 0;
    std::vector<LevelDev> L;
    mrs_comm* comm = nullptr;  // multi-GPU: NCCL communicator (dist = set)
    bool dist = false;
    int overlap = 1;           // halo exchange overlapped with interior rows (knob)
    cudaStream_t cstream = nullptr;            // communication stream (dist)
    cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
    double* inv = nullptr;
    int64_t nc = 0;
    const int* body_guard = nullptr;   // capture of unrolled loop-body copies (&st->stop)
    int dense_from = -1;       // collapsed V-cycle tail: level, dense operator, rows
    double* tail_op = nullptr;
    int64_t tail_n = 0;
    std::vector<void*> owned;
    // Krylov workspace
    double *B = nullptr, *X = nullptr, *r = nullptr, *r0 = nullptr, *p = nullptr, *q = nullptr;
    double *v = nullptr, *s = nullptr, *t = nullptr, *ph = nullptr, *sh = nullptr, *z = nullptr,
           *zt = nullptr;
    // PBiCGStab only: r_init, accumulated correction, w, y, drift-check vector,
    // second preconditioner scratch pair
    double *rinit = nullptr, *zacc = nullptr, *w = nullptr, *yv = nullptr, *chk = nullptr,
           *pa = nullptr, *pb = nullptr;
    // device state + reduction scratch
    SolveState* st = nullptr;
    double* history = nullptr;
    double* partials = nullptr;
    unsigned int* ticket = nullptr;
    double* red_out = nullptr;
    bool finalized = false;
    // whole-solve graphs, one per (x_is_zero, bound B, bound X): the plan's
    // own B/X buffers (host or staged inputs) or a caller's device buffers
    // bound in place (single GPU: no halo rows on level-0 vectors)
    struct BoundGraph {
        int gi;
        const double* B;
        double* X;
        cudaGraph_t g;
        cudaGraphExec_t e;
    };
    std::vector<BoundGraph> graphs;
    double* own_B = nullptr;   // the plan's staging buffers (B, X hold the bound ones
    double* own_X = nullptr;   // while a bound graph is captured)
    SolveState* st_host = nullptr;   // pinned copies read back after a solve
    double* hist_host = nullptr;
    // exec mode 2: one captured body graph per iteration, host-checked stop
    cudaGraph_t body_graph[2] = {nullptr, nullptr};
    cudaGraphExec_t body_exec[2] = {nullptr, nullptr};
    std::vector<std::function<cudaError_t(cudaStream_t)>> pro_list[2], epi_list[2];
    int* stop_host = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int body_kernels = 0;
    int fixed_kernels = 0;
    double it_bytes = 0;
    ~mrs_plan() {
        for (auto& bg : graphs) {
            cudaGraphExecDestroy(bg.e);
            cudaGraphDestroy(bg.g);
        }
        if (st_host) cudaFreeHost(st_host);
        if (hist_host) cudaFreeHost(hist_host);
        for (int i = 0; i < 2; ++i) {
            if (body_exec[i]) cudaGraphExecDestroy(body_exec[i]);
            if (body_graph[i]) cudaGraphDestroy(body_graph[i]);
        }
        if (stop_host) cudaFreeHost(stop_host);
        if (cstream) cudaStreamDestroy(cstream);
        if (ev_pack) cudaEventDestroy(ev_pack);
        if (ev_comm) cudaEventDestroy(ev_comm);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (void* p : owned) cudaFree(p);
    }
};

namespace {

// ---------------------------------------------------------------------------
// schedule builder
// ---------------------------------------------------------------------------

// Where the zero-guess first smoother step of a level lands (see spmm.cuh
// seed_value): the producer of the level's right-hand side writes it.
struct Seed {
    int mode = 0;             // 0 none, 1 Jacobi w*(b/d), 2 Chebyshev b/(d*theta)
    double* out = nullptr;
    const double* d = nullptr;
    double w = 0.0;           // Jacobi weight or Chebyshev theta
};

struct XB { double* cur; double* alt; void swap() { std::swap(cur, alt); } };

struct Builder {
    mrs_plan* P;
    std::vector<Launch>* out;
    const int* guard = nullptr;       // body kernels: &st->skip
    double bytes = 0;                 // algorithmic bytes accumulated
    int kernels = 0;
    double V(int64_t rows, bool f32 = false) const { return (double)rows * P->m * (f32 ? 4.0 : 8.0); }
    // vector precision of a launch gathering level-precision gx and writing gy
    static int vp(bool gx32, bool gy32) {
        return gx32 ? (gy32 ? VP_FF : VP_FD) : (gy32 ? VP_DF : VP_DD);
    }

    RedArgs red(int epi) const {
        RedArgs r;
        r.partials = P->partials; r.ticket = P->ticket; r.out = P->red_out;
        r.st = P->st; r.epi = epi;
        return r;
    }
    static SpArgs sp0() { SpArgs a; memset(&a, 0, sizeof(a)); return a; }
    static VArgs v0() { VArgs a; memset(&a, 0, sizeof(a)); return a; }

    // multi-GPU: exchange the halo rows of a gathered operand before its use
    void exchange(const Halo* h, const double* x) {
        // (the test-only loopback transport joins every exchange, active or not:
        // its collectives are barriers of all ranks)
        if (!P->dist || !h || (!h->active() && !P->comm->loop)) return;
        const Halo* hh = h;
        const mrs_comm* c = P->comm;
        const int64_t m = P->m;
        double* xx = const_cast<double*>(x);
        const int* g = guard;
        out->push_back([=](cudaStream_t s) { return halo_exchange(*hh, xx, m, c, g, s); });
    }
    // multi-GPU: a reduction finishes as local partials (kernel, EPI_NONE) ->
    // ncclAllReduce -> epilogue kernel.  Returns the epilogue to run in-kernel.
    int split_reduction(RedArgs& r) {
        if (!P->dist || r.epi == EPI_NONE) return r.epi;
        const int epi = r.epi;
        r.epi = EPI_NONE;
        return -epi - 1;   // marker: post-kernel allreduce + epilogue needed
    }
    void post_reduction(int marker, int Km, int nsets = 1) {
        if (marker >= 0) return;
        const int epi = -marker - 1;
        double* buf = P->red_out;
        const mrs_comm* c = P->comm;
        SolveState* st = P->st;
        const int m = (int)P->m;
        const int* g = guard;
        out->push_back([=](cudaStream_t s) { return allreduce_sum(buf, nsets * Km, c, s); });
        out->push_back([=](cudaStream_t s) {
            return launch_epilogue(st, buf, Km, m, epi, g, s, nsets);
        });
    }
    // multi-GPU with halo/compute overlap: the rows that read no halo column
    // run while the exchange is in flight on the plan's communication stream
    // (knob halo_overlap: 0 off, 1 on, 2 = test mode: every product with an
    // interior range, with or without a halo, whatever its size)
    bool overlapped(const DevCsr& A) const {
        const Halo* h = A.halo;
        if (!P->dist || P->overlap == 0 || !h) return false;
        if (P->overlap == 1 && !(h->active() || P->comm->loop)) return false;
        const int64_t min_rows = P->overlap == 2 ? 1 : kMinOverlapRows;
        if (A.n_long) return false;          // long-row CTAs index absolute rows
        const auto [ilo, ihi] = interior(A);
        return ihi - ilo >= min_rows && ihi <= A.nrows;
    }
    // the interior range rounded inward to slab boundaries (split launches
    // start on a slab: their slab-base table is offset, not re-indexed)
    static std::pair<int64_t, int64_t> interior(const DevCsr& A) {
        int64_t ilo = A.halo->ilo, ihi = A.halo->ihi;
        if (A.slab_base) {
            const int64_t q = 1ll << A.slab_shift;
            ilo = (ilo + q - 1) / q * q;
            ihi = ihi / q * q;
            if (ihi < ilo) ihi = ilo;
        }
        return {ilo, ihi};
    }
    // A fused dot of a distributed SpMM leaves kDotSets partial sets (one per
    // launch of a split product, empty sets zeroed), on every rank whether or
    // not its own product splits; the epilogue sums them in set order.
    static constexpr int kDotSets = 3;
    void zero_sets(int first, int last) {           // partial sets [first, last)
        if (first >= last) return;
        double* p0 = P->red_out + (int64_t)first * P->m;
        const size_t nb = sizeof(double) * (size_t)(last - first) * P->m;
        out->push_back([=](cudaStream_t s) { return cudaMemsetAsync(p0, 0, nb, s); });
    }
    void spmm(int op, const DevCsr& A, SpArgs a, double extra_bytes) {
        a.guard = guard;
        int64_t m = P->m;
        if (overlapped(A)) {
            spmm_overlapped(op, A, a);
        } else {
            exchange(A.halo, a.x);
            const int mk = a.dot ? split_reduction(a.red) : 0;
            out->push_back([=](cudaStream_t s) { return launch_spmm(op, A, a, m, s); });
            if (a.dot && mk < 0 && P->overlap) {
                zero_sets(1, kDotSets);                 // the shape of a split product
                post_reduction(mk, (int)m, kDotSets);
            } else if (a.dot) {
                post_reduction(mk, (int)m);
            }
            kernels++;
        }
        bytes += A.bytes() + extra_bytes;
    }
    // pack (compute stream) -> transfer (comm stream) || interior rows
    // [ilo, ihi) (compute stream) -> join -> boundary rows [0, ilo) and
    // [ihi, n).  Every row is computed by exactly one launch in its own entry
    // order: results are those of the unsplit product.
    void spmm_overlapped(int op, const DevCsr& A, SpArgs a) {
        const Halo* h = A.halo;
        const mrs_comm* c = P->comm;
        const int64_t m = P->m;
        double* xx = const_cast<double*>(a.x);
        const int* g = guard;
        cudaStream_t cs = P->cstream;
        cudaEvent_t ev_pack = P->ev_pack, ev_comm = P->ev_comm;
        out->push_back([=](cudaStream_t s) -> cudaError_t {
            cudaError_t e = halo_pack(*h, xx, m, g, s);
            if (e == cudaSuccess) e = cudaEventRecord(ev_pack, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev_pack, 0);
            if (e == cudaSuccess) e = halo_transfer(*h, xx, m, c, cs);
            if (e == cudaSuccess) e = cudaEventRecord(ev_comm, cs);
            return e;
        });
        const int mk = a.dot ? split_reduction(a.red) : 0;
        const auto [ilo, ihi] = interior(A);
        const int64_t n = A.nrows;
        const int64_t range[3][2] = {{ilo, ihi}, {0, ilo}, {ihi, n}};
        int last = 0;                                     // the last launch takes the long rows
        for (int k = 0; k < 3; ++k)
            if (range[k][1] > range[k][0]) last = k;
        for (int k = 0; k < 3; ++k) {
            if (k == 1)                                   // boundary rows need the halo
                out->push_back([=](cudaStream_t s) { return cudaStreamWaitEvent(s, ev_comm, 0); });
            const int64_t r0 = range[k][0], r1 = range[k][1];
            if (r1 <= r0) {
                if (a.dot && mk < 0) zero_sets(k, k + 1);
                continue;
            }
            SpArgs ak = a;
            ak.row0 = r0;
            ak.vrows = r1 - r0;
            ak.no_long_ctas = k != last;
            if (a.dot) ak.red.out = a.red.out + k * m;    // partial set k
            out->push_back([=](cudaStream_t s) { return launch_spmm(op, A, ak, m, s); });
            kernels++;
        }
        if (a.dot) post_reduction(mk, (int)m, kDotSets);
    }
    void vec(int op, VArgs a, double b) {
        a.guard = a.guard ? a.guard : guard;
        a.m = P->m;
        const int K = vec_op_k(op);
        const int mk = K ? split_reduction(a.red) : 0;
        out->push_back([=](cudaStream_t s) { return launch_vec(op, a, s); });
        if (K) post_reduction(mk, K * (int)P->m);
        bytes += b;
        kernels++;
    }
    static void set_seed(VArgs& a, const Seed& sd) {
        a.seed = sd.mode; a.seed_out = sd.out; a.seed_d = sd.d; a.seed_w = sd.w;
    }
    double seed_bytes(const Seed& sd, int64_t n) const {
        return sd.mode ? V(n) + 8.0 * n : 0.0;
    }

    // y = A x (mode); optional fused dot (dvec or x own row) . y -> epilogue;
    // optional seed of y for the level whose diagonal is sd.d.
    void spmv(const DevCsr& A, const double* x, double* y, int mode, const double* b = nullptr,
              int dot_epi = -1, const double* dvec = nullptr, const Seed& sd = Seed(),
              int vprec = VP_DD) {
        SpArgs a = sp0();
        a.x = x; a.y = y; a.b = b; a.mode = mode; a.vp = vprec;
        const bool x32 = vprec == VP_FF || vprec == VP_FD, y32 = vprec == VP_FF || vprec == VP_DF;
        double vb = V(A.ncols, x32) + V(A.nrows, y32) +
                    (mode == MRS_MODE_ASSIGN ? 0 : V(A.nrows, y32));
        if (dot_epi >= 0) {
            a.dot = 1; a.red = red(dot_epi); a.x_in = dvec; vb += V(A.nrows);
        }
        if (sd.mode) {
            a.seed = sd.mode; a.seed_out = sd.out; a.d = sd.d;
            if (sd.mode == 1) a.w = sd.w; else a.theta = sd.w;
            vb += sd.mode ? V(A.nrows, y32) + 8.0 * A.nrows : 0.0;
        }
        spmm(OP_SPMV, A, a, vb);
    }
    void dot(const double* x, const double* y, int64_t n, int epi) {
        VArgs a = v0(); a.n = n; a.x = x; a.z = y; a.red = red(epi);
        vec(V_DOT, a, 2 * V(n));
    }
    void copy(const double* x, double* y, int64_t n, const Seed& sd = Seed()) {
        VArgs a = v0(); a.n = n; a.x = x; a.y = y; set_seed(a, sd);
        vec(V_COPY, a, 2 * V(n) + seed_bytes(sd, n));
    }
    void seed_kernel(const double* b, int64_t n, const Seed& sd) {
        VArgs a = v0(); a.n = n; a.x = b; a.y = sd.out; set_seed(a, sd);
        vec(V_SEED, a, 2 * V(n) + 8.0 * n);
    }

    // ---- smoothers -----------------------------------------------------
    static bool coarsest(const mrs_plan& p, int l) {
        return p.desc.precond == MRS_PC_MG && l == (int)p.L.size() - 1;
    }
    // the collapsed sub-V-cycle (mrs_plan_set_dense_tail): entered with zero x
    static bool dense_tail(const mrs_plan& p, int l) {
        // distributed plans: only where the level is replicated (agglomerated)
        return p.desc.precond == MRS_PC_MG && l == p.dense_from &&
               (!p.dist || p.L[l].replicated);
    }

    // Gauss-Seidel sweep in place on x (blas2.py:113-162): forward and/or
    // backward half, each one cluster launch over the level schedule.
    void sgs_sweep(LevelDev& lv, const double* b, double* x, int direction) {
        const int64_t n = lv.A.nrows;
        for (int h = 0; h < 2; ++h) {
            if ((h == 0 && direction == MRS_SGS_BACKWARD) || (h == 1 && direction == MRS_SGS_FORWARD))
                continue;
            SgsArgs a;
            memset(&a, 0, sizeof(a));
            a.rp = lv.A.rp; a.ci = lv.A.ci; a.vals = lv.A.v;
            a.slab_base = lv.A.slab_base; a.slab_shift = lv.A.slab_shift;
            a.meta = lv.sgs_meta[h]; a.lptr = lv.sgs_lptr[h]; a.nlev = lv.sgs_nlev[h];
            a.d = lv.d; a.b = b; a.x = x; a.m = (int)P->m; a.guard = guard;
            a.nrows = (int)n;
            const int vb = lv.A.vb, ib = lv.A.ib;
            out->push_back([=](cudaStream_t s) { return launch_sgs(a, vb, ib, s); });
            bytes += lv.A.bytes() + 3 * V(n) + 16.0 * n;
            kernels++;
        }
    }

    // Seed a level needs when entered with a zero x (buffers of x given).
    Seed level_seed(int l, const XB& x) const {
        const mrs_plan& p = *P;
        Seed sd;
        if (coarsest(p, l) || dense_tail(p, l)) return sd;
        const LevelDev& lv = p.L[l];
        const mrs_smoother sm = pc_smoother(p.desc);
        sd.d = lv.d;
        if (sm.kind == MRS_SMOOTH_SGS) {
            sd.mode = 3; sd.out = x.cur;            // Gauss-Seidel starts from x = 0
        } else if (sm.kind == MRS_SMOOTH_JACOBI) {
            sd.mode = 1; sd.out = x.cur; sd.w = sm.weight;
        } else {
            sd.mode = 2; sd.w = 0.5 * (lv.lmax + lv.lmin);
            sd.out = sm.order <= 1 ? x.cur : lv.dva;
        }
        return sd;
    }

    void jacobi_sweep(LevelDev& lv, const double* b, double w, XB& x, int dot_epi) {
        SpArgs a = sp0(); a.x = x.cur; a.b = b; a.d = lv.d; a.w = w; a.x_out = x.alt;
        a.vp = lv.f32 ? VP_FF : VP_DD;
        // x gathered (ncols) + b + x_out (rows) + d
        double eb = V(lv.A.ncols, lv.f32) + 2 * V(lv.A.nrows, lv.f32) + 8.0 * lv.A.nrows;
        if (dot_epi >= 0) { a.dot = 1; a.red = red(dot_epi); }
        spmm(OP_JAC_SWEEP, lv.A, a, eb);
        x.swap();
    }

    // Chebyshev recurrence steps k0..order-1 (solvers.py:559-571); dv_cur holds dv.
    void cheb_steps(LevelDev& lv, const double* b, int order, int k0, double rho,
                    const double* r_in, const double* x_in, double* dv_cur, double* dv_alt,
                    XB& x, int dot_epi) {
        const double lmin = lv.lmin, lmax = lv.lmax;
        const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
        const double sigma = theta / delta;
        const int64_t n = lv.A.nrows;
        for (int k = k0; k < order; ++k) {
            const double rho_new = 1.0 / (2.0 * sigma - rho);
            SpArgs a = sp0(); a.x = dv_cur; a.x_in = x_in; a.r_in = r_in; a.d = lv.d; a.b = b;
            a.c1 = rho_new * rho; a.c2 = 2.0 * rho_new / delta;
            a.x_out = x.cur;
            a.vp = lv.f32 ? VP_FF : VP_DD;
            const bool more = k + 1 < order;
            a.r_out = more ? lv.r : nullptr;
            a.dv_out = more ? dv_alt : nullptr;
            const bool f = lv.f32;
            double eb = 4 * V(n, f) + 8.0 * n + (more ? 2 * V(n, f) : 0);
            if (!more && dot_epi >= 0) { a.dot = 1; a.red = red(dot_epi); eb += V(n, f); }
            spmm(OP_CHEB_STEP, lv.A, a, eb);
            rho = rho_new;
            std::swap(dv_cur, dv_alt);
            r_in = lv.r;
            x_in = x.cur;
        }
    }

    // The smoother a level-0 sweep preconditioner applies, or the MG pre-smoother.
    static mrs_smoother pc_smoother(const mrs_plan_desc& d) {
        if (d.precond == MRS_PC_JACOBI) return mrs_smoother{MRS_SMOOTH_JACOBI, d.pc_sweeps, d.pc_weight, 0, 0};
        if (d.precond == MRS_PC_SGS) return mrs_smoother{MRS_SMOOTH_SGS, d.pc_sweeps, 0.0, 0, d.pc_direction};
        return d.pre;   // MultiGrid pre-smoother; Chebyshev preconditioner (pre.order)
    }

    // Smoother on a NONZERO x (post-smoothing; pre-smoothing of later cycles).
    void smooth_nonzero(LevelDev& lv, const double* b, const mrs_smoother& sm, XB& x, int dot_epi) {
        const int64_t n = lv.A.nrows;
        if (sm.kind == MRS_SMOOTH_SGS) {
            const int sweeps = sm.sweeps < 1 ? 1 : sm.sweeps;
            for (int k = 0; k < sweeps; ++k) sgs_sweep(lv, b, x.cur, sm.direction);
            if (dot_epi >= 0) dot(b, x.cur, n, dot_epi);
            return;
        }
        if (sm.kind == MRS_SMOOTH_JACOBI) {
            if (sm.weight == 0.0) {          // blas2.py:487-489: no-op
                if (dot_epi >= 0) dot(b, x.cur, n, dot_epi);
                return;
            }
            const int sweeps = sm.sweeps < 1 ? 1 : sm.sweeps;
            for (int k = 0; k < sweeps; ++k)
                jacobi_sweep(lv, b, sm.weight, x, k == sweeps - 1 ? dot_epi : -1);
            return;
        }
        const int order = sm.order < 1 ? 1 : sm.order;
        const double theta = 0.5 * (lv.lmax + lv.lmin), delta = 0.5 * (lv.lmax - lv.lmin);
        SpArgs a = sp0(); a.x = x.cur; a.b = b; a.d = lv.d; a.theta = theta;
        a.x_out = x.alt;
        a.vp = lv.f32 ? VP_FF : VP_DD;
        const bool more = order > 1;
        a.r_out = more ? lv.r : nullptr;
        a.dv_out = more ? lv.dva : nullptr;
        const bool f = lv.f32;
        double eb = 3 * V(n, f) + 8.0 * n + (more ? 2 * V(n, f) : 0);
        if (!more && dot_epi >= 0) { a.dot = 1; a.red = red(dot_epi); }
        spmm(OP_CHEB_FIRST, lv.A, a, eb);
        x.swap();
        if (more)
            cheb_steps(lv, b, order, 1, 1.0 / (theta / delta), lv.r, x.cur, lv.dva, lv.dvb, x,
                       dot_epi);
    }

    // Pre-smoother on a ZERO x whose seed is already in place (level_seed).
    void smooth_zero_seeded(LevelDev& lv, const double* b, const mrs_smoother& sm, XB& x,
                            int dot_epi) {
        const int64_t n = lv.A.nrows;
        if (sm.kind == MRS_SMOOTH_SGS) {                 // x.cur = 0 (seed mode 3)
            smooth_nonzero(lv, b, sm, x, dot_epi);
            return;
        }
        if (sm.kind == MRS_SMOOTH_JACOBI) {
            const int sweeps = sm.sweeps < 1 ? 1 : sm.sweeps;
            if (sm.weight != 0.0)
                for (int k = 1; k < sweeps; ++k)
                    jacobi_sweep(lv, b, sm.weight, x, k == sweeps - 1 ? dot_epi : -1);
            if ((sweeps == 1 || sm.weight == 0.0) && dot_epi >= 0) dot(b, x.cur, n, dot_epi);
            return;
        }
        const int order = sm.order < 1 ? 1 : sm.order;
        if (order == 1) {                    // x = dv0 = b/(d*theta)
            if (dot_epi >= 0) dot(b, x.cur, n, dot_epi);
            return;
        }
        const double theta = 0.5 * (lv.lmax + lv.lmin), delta = 0.5 * (lv.lmax - lv.lmin);
        // after the first step: x = dv0 (in lv.dva), r = b
        cheb_steps(lv, b, order, 1, 1.0 / (theta / delta), b, lv.dva, lv.dva, lv.dvb, x, dot_epi);
    }

    // V-cycle on level l (solvers.py:651-664).  zero: x certified zero and its
    // seed already written by the producer of b (seeded) or by a seed kernel.
    void vcycle(int l, const double* b, bool zero, bool seeded, XB& x, int dot_epi) {
        mrs_plan& p = *P;
        LevelDev& lv = p.L[l];
        if (coarsest(p, l) || (zero && dense_tail(p, l))) {
            // x = A_c^{-1} b (replaces the LU solve, solvers.py:644-649), or
            // x = T_l b for the collapsed tail (same dense kernel)
            const bool tl = !coarsest(p, l);
            int64_t m = p.m, nc = tl ? p.tail_n : p.nc;
            const double* inv = tl ? p.tail_op : p.inv;
            double* xo = x.cur;
            const int* g = guard;
            if (tl)
                out->push_back([=](cudaStream_t s) { return launch_dense(inv, nc, b, xo, m, g, s); });
            else
                out->push_back([=](cudaStream_t s) { return launch_coarse(inv, nc, b, xo, m, g, s); });
            bytes += (double)nc * nc * 8.0 + 2 * V(nc);
            kernels++;
            if (dot_epi >= 0) dot(b, x.cur, nc, dot_epi);
            return;
        }
        const mrs_smoother& pre = p.desc.pre;
        if (zero) {
            if (!seeded) seed_kernel(b, lv.A.nrows, level_seed(l, x));
            smooth_zero_seeded(lv, b, pre, x, -1);
        } else {
            smooth_nonzero(lv, b, pre, x, -1);
        }
        LevelDev& lc = p.L[l + 1];
        spmv(lv.A, x.cur, lv.r, MRS_MODE_RSUB, b, -1, nullptr, Seed(),
             vp(lv.f32, lv.f32));                                      // r = b - A x
        XB xc{lc.xa, lc.xb};
        if (p.dist && lc.replicated && !lv.replicated) {
            // agglomeration: my slice of rc = R r, allgather, replicated below
            spmv(lv.R, lv.r, lc.b + lc.slice_row0 * p.m, MRS_MODE_ASSIGN);
            double* buf = lc.b;
            const int64_t cnt = lc.slice_rows * p.m;
            const mrs_comm* c = p.comm;
            out->push_back([=](cudaStream_t s) { return allgather_inplace(buf, cnt, c, s); });
            vcycle(l + 1, lc.b, true, false, xc, -1);
        } else {
            spmv(lv.R, lv.r, lc.b, MRS_MODE_ASSIGN, nullptr, -1, nullptr,
                 level_seed(l + 1, xc), vp(lv.f32, lc.f32));          // rc = R r (+ seed)
            vcycle(l + 1, lc.b, true, true, xc, -1);
        }
        spmv(lv.P, xc.cur, x.cur, MRS_MODE_ADD, nullptr, -1, nullptr, Seed(),
             vp(lc.f32, lv.f32));                                      // x += P xc
        smooth_nonzero(lv, b, p.desc.post, x, dot_epi);
    }
};

// A planned preconditioner application z = M r at level 0.
struct PCPlan {
    std::vector<Launch> ops;
    double* out = nullptr;     // buffer holding z
    Seed seed;                 // level-0 seed the producer of r must write
    double bytes = 0;
    int kernels = 0;
};

// Build z = M r into `want` (buffers want/spare).  producer_seeds: the kernel
// producing r also writes the level-0 seed (plan.seed); otherwise a seed
// kernel is emitted.  dot_epi >= 0: the last kernel also reduces (r, z).
PCPlan plan_precond(mrs_plan* P, const int* guard, const double* r, double* want,
                    double* spare, bool producer_seeds, int dot_epi) {
    const mrs_plan_desc& d = P->desc;
    auto build = [&](double* a, double* b, PCPlan& pc) {
        Builder bd{P, &pc.ops, guard};
        XB x{a, b};
        if (d.precond == MRS_PC_NONE) {
            pc.out = const_cast<double*>(r);
            if (dot_epi >= 0) bd.dot(r, r, P->n, dot_epi);
        } else if (d.precond == MRS_PC_JACOBI || d.precond == MRS_PC_SGS ||
                   d.precond == MRS_PC_CHEB) {
            LevelDev& lv = P->L[0];
            pc.seed = bd.level_seed(0, x);
            if (!producer_seeds) bd.seed_kernel(r, P->n, pc.seed);
            bd.smooth_zero_seeded(lv, r, Builder::pc_smoother(d), x, dot_epi);
            pc.out = x.cur;
        } else if (P->L[0].f32) {
            // fp32 preconditioner (vec32 = 2): the whole V-cycle, level 0 included,
            // on float vectors; r -> float b (+ seed) on entry, float x -> z on exit
            const int cycles = d.mg_cycles < 1 ? 1 : d.mg_cycles;
            LevelDev& lv = P->L[0];
            XB x32{lv.xa, lv.xb};
            const Seed sd = bd.level_seed(0, x32);
            const int64_t n = P->n, m = P->m;
            {
                const double* rr = r;
                float* b32 = reinterpret_cast<float*>(lv.b);
                float* so = reinterpret_cast<float*>(sd.out);
                const int md = sd.mode;
                const double* dd = sd.d;
                const double w = sd.w;
                const int* g = guard;
                pc.ops.push_back([=](cudaStream_t s) {
                    return launch_cvt_to32(rr, b32, n, m, md, dd, w, so, g, s);
                });
                bd.bytes += bd.V(n) + bd.V(n, true) * (md ? 2 : 1) + (md ? 8.0 * n : 0.0);
                bd.kernels++;
            }
            for (int c = 0; c < cycles; ++c) bd.vcycle(0, lv.b, c == 0, c == 0, x32, -1);
            {
                const float* xs = reinterpret_cast<const float*>(x32.cur);
                double* z = a;
                const int* g = guard;
                pc.ops.push_back([=](cudaStream_t s) { return launch_cvt_from32(xs, z, n * m, g, s); });
                bd.bytes += bd.V(n) + bd.V(n, true);
                bd.kernels++;
            }
            if (dot_epi >= 0) bd.dot(r, a, n, dot_epi);
            pc.out = a;
            pc.seed = Seed();
            pc.bytes = bd.bytes;
            pc.kernels = bd.kernels;
            return;
        } else {
            const int cycles = d.mg_cycles < 1 ? 1 : d.mg_cycles;
            pc.seed = bd.level_seed(0, x);
            for (int c = 0; c < cycles; ++c)
                bd.vcycle(0, r, c == 0, c == 0 && producer_seeds, x,
                          c == cycles - 1 ? dot_epi : -1);
            pc.out = x.cur;
        }
        if (!producer_seeds) pc.seed = Seed();
        pc.bytes = bd.bytes;
        pc.kernels = bd.kernels;
    };
    PCPlan dry;
    build(want, spare, dry);
    if (dry.out == spare) std::swap(want, spare);
    PCPlan pc;
    build(want, spare, pc);
    return pc;
}

// ---------------------------------------------------------------------------
// drivers
// ---------------------------------------------------------------------------

struct Program {
    std::vector<Launch> pro, body, epi;
    double body_bytes = 0;
    int body_kernels = 0;
};

void append(std::vector<Launch>& dst, std::vector<Launch>& src) {
    dst.insert(dst.end(), src.begin(), src.end());
}

void build_cg(mrs_plan* P, bool x_zero, Program& pg) {
    const int64_t n = P->n;
    // unrolled body copies are guarded by `stop` (skip implies stop)
    const int* skip = P->body_guard ? P->body_guard : &P->st->skip;
    const DevCsr& A = P->L[0].A;
    const mrs_plan_desc& d = P->desc;
    const bool pc_on = d.precond != MRS_PC_NONE;
    // prologue (solvers.py:156-168)
    {
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        PCPlan pc = plan_precond(P, nullptr, P->r, P->z, P->zt, pc_on, EPI_RHO);
        if (x_zero) b.copy(P->B, P->r, n, pc.seed);
        else b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B, -1, nullptr, pc.seed);
        b.dot(P->r, P->r, n, EPI_RNORM_INIT);
        append(pg.pro, pc.ops);
        b.copy(pc.out, P->p, n);
    }
    // body (solvers.py:171-186)
    {
        Builder b{P, &pg.body, skip};
        b.spmv(A, P->p, P->q, MRS_MODE_ASSIGN, nullptr, EPI_CG_ALPHA);   // q = A p ; alpha
        const bool jac1 = d.precond == MRS_PC_JACOBI && d.pc_sweeps <= 1;
        double* z;
        if (jac1) {
            // X += a p ; r -= a q ; z = w r/d ; (r.r, r.z) -> rnorm, beta
            VArgs a = Builder::v0(); a.n = n; a.y = P->X; a.x = P->p; a.y2 = P->r; a.u = P->q;
            a.a = P->st->alpha; a.b = P->st->neg_alpha; a.y3 = P->z; a.d = P->L[0].d;
            a.wt = d.pc_weight; a.red = b.red(EPI_CG_RNORM_BETA);
            b.vec(V_CG_UPDATE_JAC, a, 6 * b.V(n) + 8.0 * n);
            z = P->z;
        } else {
            PCPlan pc = plan_precond(P, skip, P->r, P->z, P->zt, pc_on,
                                     pc_on ? EPI_CG_BETA : -1);
            VArgs a = Builder::v0(); a.n = n; a.y = P->X; a.x = P->p; a.y2 = P->r; a.u = P->q;
            a.a = P->st->alpha; a.b = P->st->neg_alpha;
            a.red = b.red(pc_on ? EPI_CG_RNORM : EPI_CG_RNORM_BETA1);
            Builder::set_seed(a, pc.seed);
            b.vec(V_CG_UPDATE, a, 5 * b.V(n) + b.seed_bytes(pc.seed, n));
            append(pg.body, pc.ops);
            b.bytes += pc.bytes; b.kernels += pc.kernels;
            z = pc.out;
        }
        VArgs pu = Builder::v0(); pu.n = n; pu.y = P->p; pu.x = z; pu.b = P->st->beta;
        b.vec(V_P_UPDATE, pu, 3 * b.V(n));
        pg.body_bytes = b.bytes;
        pg.body_kernels = b.kernels;
    }
    // true residual (solvers.py:126-141)
    {
        Builder b{P, &pg.epi, nullptr};
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

void build_bicgstab(mrs_plan* P, bool x_zero, Program& pg) {
    const int64_t n = P->n;
    const int* skip = &P->st->skip;
    const DevCsr& A = P->L[0].A;
    const bool pc_on = P->desc.precond != MRS_PC_NONE;
    PCPlan pph = plan_precond(P, skip, P->p, P->ph, P->zt, pc_on, -1);
    PCPlan psh = plan_precond(P, skip, P->s, P->sh, P->zt, pc_on, -1);
    // prologue (solvers.py:220-243 and the first-iteration rho, p = r)
    {
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        if (x_zero) b.copy(P->B, P->r, n);
        else b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.copy(P->r, P->r0, n);
        b.dot(P->r, P->r, n, EPI_RNORM_INIT);
        b.dot(P->r0, P->r, n, EPI_RHO);
        b.copy(P->r, P->p, n, pph.seed);       // p = r, and the seed for ph = M p
    }
    {
        Builder b{P, &pg.body, skip};
        // p = r + beta (p - omega v)  -- not in the first iteration (it == 0)
        VArgs pu = Builder::v0(); pu.n = n; pu.y = P->p; pu.x = P->r; pu.v = P->v;
        pu.b = P->st->beta; pu.c = P->st->neg_omega; pu.guard_it = &P->st->it;
        Builder::set_seed(pu, pph.seed);
        b.vec(V_BICG_P, pu, 4 * b.V(n) + b.seed_bytes(pph.seed, n));
        const double* ph = pc_on ? pph.out : P->p;
        append(pg.body, pph.ops);
        b.bytes += pph.bytes; b.kernels += pph.kernels;
        b.spmv(A, ph, P->v, MRS_MODE_ASSIGN, nullptr, EPI_BICG_ALPHA, P->r0);  // v = A ph; (r0, v)
        VArgs sa = Builder::v0(); sa.n = n; sa.y = P->s; sa.x = P->r; sa.v = P->v;
        sa.a = P->st->neg_alpha;
        Builder::set_seed(sa, psh.seed);
        b.vec(V_BICG_S, sa, 3 * b.V(n) + b.seed_bytes(psh.seed, n));      // s = r - alpha v
        const double* sh = pc_on ? psh.out : P->s;
        append(pg.body, psh.ops);
        b.bytes += psh.bytes; b.kernels += psh.kernels;
        b.spmv(A, sh, P->t, MRS_MODE_ASSIGN);                              // t = A sh
        VArgs d3 = Builder::v0(); d3.n = n; d3.x = P->t; d3.s = P->s; d3.red = b.red(EPI_BICG_OMEGA);
        b.vec(V_DOT3, d3, 2 * b.V(n));                                     // omega
        VArgs xr = Builder::v0(); xr.n = n; xr.y = P->X; xr.u = ph; xr.v = sh; xr.s = P->s;
        xr.w = P->t; xr.y2 = P->r; xr.z = P->r0;
        xr.a = P->st->alpha; xr.b = P->st->omega; xr.c = P->st->neg_omega;
        xr.red = b.red(EPI_BICG_RNORM);
        b.vec(V_BICG_XR, xr, 8 * b.V(n));                                  // X, r, (r0,r), (r,r)
        pg.body_bytes = b.bytes;
        pg.body_kernels = b.kernels;
    }
    {
        Builder b{P, &pg.epi, nullptr};
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

// Reordered BiCGStab (solvers.py:296-364): two reduction groups per
// iteration; rho' and ||r'|| come from the linear relations
// rho' = (r0,s) - omega (r0,t), ||r'||^2 = (s,s) - 2 omega (t,s) + omega^2 (t,t).
// merged=1 is bitwise identical here (paired_update == add2_scaled + axpby).
void build_rbicgstab(mrs_plan* P, bool x_zero, Program& pg) {
    const int64_t n = P->n;
    SolveState* st = P->st;
    const int* skip = &st->skip;
    const DevCsr& A = P->L[0].A;
    const bool pc_on = P->desc.precond != MRS_PC_NONE;
    PCPlan pph = plan_precond(P, skip, P->p, P->ph, P->zt, pc_on, -1);
    PCPlan psh = plan_precond(P, skip, P->s, P->sh, P->zt, pc_on, -1);
    {   // prologue (solvers.py:302-319)
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        if (x_zero) b.copy(P->B, P->r, n);
        else b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.copy(P->r, P->r0, n);
        b.dot(P->r, P->r, n, EPI_RNORM_INIT);
        b.dot(P->r0, P->r, n, EPI_RHO);
        b.copy(P->r, P->p, n, pph.seed);        // p = r (first iteration) + seed of M p
    }
    {   // body (solvers.py:322-359)
        Builder b{P, &pg.body, skip};
        const double* ph = pc_on ? pph.out : P->p;
        append(pg.body, pph.ops);
        b.bytes += pph.bytes; b.kernels += pph.kernels;
        b.spmv(A, ph, P->v, MRS_MODE_ASSIGN, nullptr, EPI_BICG_ALPHA, P->r0);  // v = A ph; (r0,v)
        VArgs sa = Builder::v0(); sa.n = n; sa.y = P->s; sa.x = P->r; sa.v = P->v;
        sa.a = st->neg_alpha;
        Builder::set_seed(sa, psh.seed);
        b.vec(V_BICG_S, sa, 3 * b.V(n) + b.seed_bytes(psh.seed, n));       // s = r - alpha v
        const double* sh = pc_on ? psh.out : P->s;
        append(pg.body, psh.ops);
        b.bytes += psh.bytes; b.kernels += psh.kernels;
        b.spmv(A, sh, P->t, MRS_MODE_ASSIGN);                               // t = A sh
        VArgs d5 = Builder::v0(); d5.n = n; d5.x = P->t; d5.s = P->s; d5.z = P->r0;
        d5.red = b.red(EPI_RBICG_OMEGA);
        b.vec(V_DOT5, d5, 3 * b.V(n));                                      // reduction group 2
        VArgs xr = Builder::v0(); xr.n = n; xr.y = P->X; xr.u = ph; xr.v = sh; xr.s = P->s;
        xr.w = P->t; xr.y2 = P->r;
        xr.a = st->alpha; xr.b = st->omega; xr.c = st->neg_omega;
        b.vec(V_BICG_XR0, xr, 7 * b.V(n));                                  // X, r
        VArgs pu = Builder::v0(); pu.n = n; pu.y = P->p; pu.x = P->r; pu.v = P->v;
        pu.b = st->beta; pu.c = st->neg_omega; pu.guard = &st->pskip;
        Builder::set_seed(pu, pph.seed);
        b.vec(V_BICG_P, pu, 4 * b.V(n) + b.seed_bytes(pph.seed, n));       // p = r + beta(p - w v)
        pg.body_bytes = b.bytes;
        pg.body_kernels = b.kernels;
    }
    {
        Builder b{P, &pg.epi, nullptr};
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

// Pipelined BiCGStab (solvers.py:367-479): the solver runs on op = A M in
// the preconditioned variable (zacc); two products and two reduction groups
// per iteration; every 20th iteration (and at convergence) the recurrence
// residual is cross-checked against r_init - op(zacc).  X += M zacc at the end.
void build_pbicgstab(mrs_plan* P, bool x_zero, Program& pg) {
    const int64_t n = P->n;
    SolveState* st = P->st;
    const int* skip = &st->skip;
    const int* nodrift = &st->nodrift;
    const DevCsr& A = P->L[0].A;
    const bool pc_on = P->desc.precond != MRS_PC_NONE;
    // preconditioner applications: consecutive ops use disjoint scratch pairs,
    // so a product seeding the next application never writes what it reads
    PCPlan pc_r = plan_precond(P, nullptr, P->r, P->ph, P->zt, pc_on, -1);
    PCPlan pc_w0 = plan_precond(P, nullptr, P->w, P->pa, P->pb, pc_on, -1);
    PCPlan pc_z = plan_precond(P, skip, P->z, P->ph, P->zt, pc_on, -1);
    PCPlan pc_w = plan_precond(P, skip, P->w, P->pa, P->pb, pc_on, -1);
    PCPlan pc_d = plan_precond(P, nodrift, P->zacc, P->ph, P->zt, false, -1);
    PCPlan pc_f = plan_precond(P, nullptr, P->zacc, P->ph, P->zt, false, -1);
    const size_t vbytes = (size_t)P->L[0].vrows * P->m * 8;
    {   // prologue (solvers.py:388-409)
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        if (x_zero) b.copy(P->B, P->rinit, n);
        else b.spmv(A, P->X, P->rinit, MRS_MODE_RSUB, P->B);
        b.copy(P->rinit, P->r, n, pc_r.seed);
        b.copy(P->rinit, P->r0, n);
        double* za = P->zacc;
        pg.pro.push_back([=](cudaStream_t s) { return cudaMemsetAsync(za, 0, vbytes, s); });
        b.dot(P->r, P->r, n, EPI_RNORM_INIT);
        append(pg.pro, pc_r.ops);
        b.spmv(A, pc_on ? pc_r.out : P->r, P->w, MRS_MODE_ASSIGN, nullptr, -1, nullptr,
               pc_w0.seed);                                                 // w = op(r)
        append(pg.pro, pc_w0.ops);
        b.spmv(A, pc_on ? pc_w0.out : P->w, P->t, MRS_MODE_ASSIGN);        // t = op(w)
        VArgs d2 = Builder::v0(); d2.n = n; d2.x = P->r0; d2.z = P->r; d2.u = P->r0; d2.v = P->w;
        d2.red = b.red(EPI_PBICG_INIT);
        b.vec(V_DOT2, d2, 3 * b.V(n));                                      // rho, alpha
        b.copy(P->r, P->p, n);                                              // first iteration:
        b.copy(P->w, P->s, n);                                              //   p, s, z = r, w, t
        b.copy(P->t, P->z, n, pc_z.seed);
    }
    {   // body (solvers.py:427-474)
        Builder b{P, &pg.body, skip};
        VArgs qy = Builder::v0(); qy.n = n;
        qy.y = P->p; qy.y2 = P->s; qy.y3 = P->z; qy.y4 = P->q; qy.y5 = P->yv;
        qy.x = P->r; qy.w = P->w; qy.u = P->t; qy.v = P->v;
        qy.a = st->neg_alpha; qy.b = st->beta; qy.c = st->neg_omega; qy.guard_it = &st->it;
        Builder::set_seed(qy, pc_z.seed);
        qy.red = b.red(EPI_PBICG_OMEGA);
        b.vec(V_PBICG_QY, qy, 12 * b.V(n) + b.seed_bytes(pc_z.seed, n));  // group 1 -> omega
        append(pg.body, pc_z.ops);
        b.bytes += pc_z.bytes; b.kernels += pc_z.kernels;
        b.spmv(A, pc_on ? pc_z.out : P->z, P->v, MRS_MODE_ASSIGN);         // v = op(z)
        VArgs xr = Builder::v0(); xr.n = n; xr.y = P->zacc; xr.u = P->p; xr.v = P->q;
        xr.s = P->q; xr.w = P->yv; xr.y2 = P->r;
        xr.a = st->alpha; xr.b = st->omega; xr.c = st->neg_omega;
        b.vec(V_BICG_XR0, xr, 6 * b.V(n));                                  // zacc, r
        VArgs wk = Builder::v0(); wk.n = n; wk.y = P->t; wk.y2 = P->w; wk.x = P->v;
        wk.u = P->yv; wk.z = P->r0; wk.v = P->r; wk.s = P->s; wk.w = P->z;
        wk.a = st->neg_alpha; wk.c = st->neg_omega;
        Builder::set_seed(wk, pc_w.seed);
        wk.red = b.red(EPI_PBICG_RHO);
        b.vec(V_PBICG_W, wk, 9 * b.V(n) + b.seed_bytes(pc_w.seed, n));     // t, w; group 2
        append(pg.body, pc_w.ops);
        b.bytes += pc_w.bytes; b.kernels += pc_w.kernels;
        b.spmv(A, pc_on ? pc_w.out : P->w, P->t, MRS_MODE_ASSIGN);         // t = op(w)
        pg.body_bytes = b.bytes;
        pg.body_kernels = b.kernels;
        // drift check (solvers.py:415-423), only when the epilogue asked for it
        Builder bd{P, &pg.body, nodrift};
        append(pg.body, pc_d.ops);
        bd.spmv(A, pc_on ? pc_d.out : P->zacc, P->chk, MRS_MODE_ASSIGN);   // chk = op(zacc)
        VArgs ud = Builder::v0(); ud.n = n; ud.y = P->chk; ud.x = P->rinit;
        ud.a = st->one; ud.b = st->neg_one; ud.red = bd.red(EPI_PBICG_DRIFT);
        bd.vec(V_UPDATE_DOT, ud, 3 * bd.V(n));                              // r_init - chk; norm
    }
    {   // X += M zacc (solvers.py:476-479), then the true residual
        Builder b{P, &pg.epi, nullptr};
        append(pg.epi, pc_f.ops);
        VArgs xu = Builder::v0(); xu.n = n; xu.y = P->X; xu.x = pc_on ? pc_f.out : P->zacc;
        xu.a = st->one; xu.b = st->one;
        b.vec(V_AXPBY, xu, 3 * b.V(n));
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

// _stationary_solve / multigrid_solve (solvers.py:962-978, :683-710): one
// step of the configured sweep (or one V-cycle) on X per iteration, then the
// TRUE residual and its norm decide convergence; the final relative residual
// is that last norm (recomputed by the epilogue from the same X).
void build_stationary(mrs_plan* P, bool x_zero, Program& pg) {
    const int64_t n = P->n;
    const DevCsr& A = P->L[0].A;
    const mrs_plan_desc& d = P->desc;
    {
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        if (x_zero) b.copy(P->B, P->r, n);
        else b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_RNORM_INIT);
    }
    {
        // guarded by skip: a no-op once a gate (exec mode 2) saw the stop flag
        Builder b{P, &pg.body, &P->st->skip};
        LevelDev& lv = P->L[0];
        // the step runs on a NONZERO x: on the zero first guess this is the
        // reference's zero-flag short-cut value (0 + w*(b/d) == w*(b/d), ...)
        XB x{P->X, P->zt};
        if (d.precond == MRS_PC_SGS) {
            b.sgs_sweep(lv, P->B, P->X, d.pc_direction);
        } else if (d.precond == MRS_PC_JACOBI) {
            if (d.pc_weight != 0.0) b.jacobi_sweep(lv, P->B, d.pc_weight, x, -1);
        } else {
            b.vcycle(0, P->B, false, false, x, -1);
        }
        if (x.cur != P->X) b.copy(x.cur, P->X, n);
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_STAT_RNORM);
        pg.body_bytes = b.bytes;
        pg.body_kernels = b.kernels;
    }
    {
        Builder b{P, &pg.epi, nullptr};
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

// direct_solve (solvers.py:588-604): X = A^-1 B with the uploaded dense
// inverse, then the relative residual; no iterations (max_iters 0).
void build_direct(mrs_plan* P, bool, Program& pg) {
    const int64_t n = P->n;
    const DevCsr& A = P->L[0].A;
    {
        Builder b{P, &pg.pro, nullptr};
        b.dot(P->B, P->B, n, EPI_BSCALE);
        b.dot(P->B, P->B, n, EPI_RNORM_INIT);     // stop = 1 (max_iters 0)
        const double* inv = P->inv;
        const double* B = P->B;
        double* X = P->X;
        const int64_t m = P->m;
        pg.pro.push_back([=](cudaStream_t s) { return launch_dense(inv, n, B, X, m, nullptr, s); });
        b.bytes += (double)n * n * 8.0 + 2 * b.V(n);
        b.kernels++;
    }
    {
        Builder b{P, &pg.epi, nullptr};
        b.spmv(A, P->X, P->r, MRS_MODE_RSUB, P->B);
        b.dot(P->r, P->r, n, EPI_FINAL);
    }
}

void build_program(mrs_plan* P, bool x_zero, Program& pg) {
    switch (P->desc.method) {
    case MRS_METHOD_STATIONARY: build_stationary(P, x_zero, pg); break;
    case MRS_METHOD_DIRECT: build_direct(P, x_zero, pg); break;
    case MRS_METHOD_CG: build_cg(P, x_zero, pg); break;
    case MRS_METHOD_BICGSTAB: build_bicgstab(P, x_zero, pg); break;
    case MRS_METHOD_RBICGSTAB: build_rbicgstab(P, x_zero, pg); break;
    default: build_pbicgstab(P, x_zero, pg); break;
    }
}

// Exec mode 2 (distributed): one host-launched graph carries kDistUnroll
// iterations; each copy starts with this gate, which turns a stop taken in
// an earlier copy into skip flags for every kernel of this copy (the host
// checks stop once per graph launch).
constexpr int kDistUnroll = 4;
__global__ void gate_kernel(SolveState* st) {
    if (st->stop) {
        st->skip = 1;
        st->pskip = 1;
        st->nodrift = 1;
    }
}

__global__ void set_cond_kernel(SolveState* st, cudaGraphConditionalHandle h, int has) {
    st->has_cond = has;
    st->cond = h;
}

cudaError_t run_list(const std::vector<Launch>& v, cudaStream_t s) {
    for (auto& f : v) {
        cudaError_t e = f(s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int capture_graph(mrs_plan* P, bool x_zero, cudaStream_t s, cudaGraph_t* out_g,
                  cudaGraphExec_t* out_e) {
    Program pg;
    build_program(P, x_zero, pg);

    cudaGraph_t g;
    MRS_CUDA_OK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    MRS_CUDA_OK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    // first node: publish this graph's handle to the epilogues
    {
        SolveState* st = P->st;
        pg.pro.insert(pg.pro.begin(), [=](cudaStream_t s) {
            set_cond_kernel<<<1, 1, 0, s>>>(st, h, 1);
            return cudaGetLastError();
        });
    }

    // 1) prologue
    cudaStream_t cs;
    MRS_CUDA_OK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    MRS_CUDA_OK(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if (run_list(pg.pro, cs) != cudaSuccess) { cudaStreamEndCapture(cs, &g); return MRS_ERR_CUDA; }
    cudaGraph_t gg;
    MRS_CUDA_OK(cudaStreamEndCapture(cs, &gg));
    // find the sink nodes of the prologue
    size_t nn = 0;
    MRS_CUDA_OK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    MRS_CUDA_OK(cudaGraphGetNodes(g, nodes.data(), &nn));
    std::vector<cudaGraphNode_t> sinks;
    for (auto nd : nodes) {
        size_t ndep = 0;
        MRS_CUDA_OK(cudaGraphNodeGetDependentNodes(nd, nullptr, &ndep));
        if (ndep == 0) sinks.push_back(nd);
    }
    // 2) WHILE node with the iteration body (none for a loop-free program)
    std::vector<cudaGraphNode_t> after = sinks;
    if (!pg.body.empty()) {
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        MRS_CUDA_OK(cudaGraphAddNode(&wnode, g, sinks.data(), sinks.size(), &cp));
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        MRS_CUDA_OK(cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        if (run_list(pg.body, cs) != cudaSuccess) { cudaStreamEndCapture(cs, &gg); return MRS_ERR_CUDA; }
        // short CG bodies: more iterations per trip of the WHILE node (each
        // trip costs ~4 us of conditional relaunch); the extra copies run
        // only while `stop` is clear, so iterations and results are unchanged
        const int copies = (P->desc.method == MRS_METHOD_CG && pg.body.size() <= 4)
                               ? (int)loop_unroll() : 1;
        for (int u = 1; u < copies; ++u) {
            P->body_guard = &P->st->stop;
            Program pg2;
            build_program(P, x_zero, pg2);
            P->body_guard = nullptr;
            if (run_list(pg2.body, cs) != cudaSuccess) { cudaStreamEndCapture(cs, &gg); return MRS_ERR_CUDA; }
        }
        MRS_CUDA_OK(cudaStreamEndCapture(cs, &gg));
        after.assign(1, wnode);
    }
    // 3) epilogue after the loop
    MRS_CUDA_OK(cudaStreamBeginCaptureToGraph(cs, g, after.data(), nullptr, after.size(),
                                              cudaStreamCaptureModeRelaxed));
    if (run_list(pg.epi, cs) != cudaSuccess) { cudaStreamEndCapture(cs, &gg); return MRS_ERR_CUDA; }
    MRS_CUDA_OK(cudaStreamEndCapture(cs, &gg));
    cudaStreamDestroy(cs);
    cudaGraphExec_t ex;
    MRS_CUDA_OK(cudaGraphInstantiate(&ex, g, 0));
    *out_g = g;
    *out_e = ex;
    return MRS_OK;
}

int upload_csr(const mrs_host_csr* h, DevCsr& d, std::vector<void*>& owned) {
    if (!h) return MRS_OK;
    if (h->nnz > INT32_MAX || h->nrows < 0) return MRS_ERR_UNSUPPORTED;
    if (h->val_bytes != 4 && h->val_bytes != 8) return MRS_ERR_ARG;
    if (h->idx_bytes != 1 && h->idx_bytes != 2 && h->idx_bytes != 4) return MRS_ERR_ARG;
    d.nrows = h->nrows; d.ncols = h->ncols; d.nnz = h->nnz;
    d.vb = h->val_bytes;
    // device index width: >= 16 bit (u8 blocks are widened; they are tiny)
    d.ib = h->idx_bytes == 1 ? 2 : h->idx_bytes;
    std::vector<int32_t> rp(h->nrows + 1);
    for (int64_t i = 0; i <= h->nrows; ++i) rp[i] = (int32_t)h->row_ptr[i];
    // pad_ bit 0: compress 32-bit columns to slab-relative 16-bit ones on the
    // device when they fit (slab.cu)
    const bool try_slab = (h->pad_ & 1) && h->idx_bytes == 4 && !h->slab_base && h->nnz > 0;
    d.rp = dalloc<int32_t>(h->nrows + 1, owned);
    d.v = dalloc<char>((size_t)h->nnz * d.vb, owned);
    if (!d.rp || !d.v) return MRS_ERR_ALLOC;
    MRS_CUDA_OK(cudaMemcpy(d.rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice));
    bool slabbed = false;
    if (try_slab) {
        uint32_t* c32 = nullptr;
        if (cudaMalloc(&c32, (size_t)h->nnz * 4) != cudaSuccess) return MRS_ERR_ALLOC;
        if (cudaMemcpy(c32, h->col_idx, (size_t)h->nnz * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaFree(c32);
            return MRS_ERR_CUDA;
        }
        uint16_t* c16 = nullptr;
        int32_t* base = nullptr;
        int shift = 0;
        int64_t ns = 0;
        const int rc = slab_compress_device(d.rp, c32, h->nrows, h->nnz, h->ncols, &c16, &base,
                                            &shift, &ns);
        if (rc < 0) { cudaFree(c32); return MRS_ERR_CUDA; }
        if (rc == 1) {
            cudaFree(c32);
            owned.push_back(c16); owned.push_back(base);
            d.ci = c16; d.ib = 2; d.slab_base = base; d.slab_shift = shift;
        } else {
            owned.push_back(c32);
            d.ci = c32;
        }
        slabbed = true;
    } else {
        d.ci = dalloc<char>((size_t)h->nnz * d.ib, owned);
        if (!d.ci) return MRS_ERR_ALLOC;
    }
    if (slabbed) {
        // columns are in place
    } else if (h->idx_bytes == 1) {
        std::vector<uint16_t> w(h->nnz);
        for (int64_t k = 0; k < h->nnz; ++k) w[k] = ((const uint8_t*)h->col_idx)[k];
        MRS_CUDA_OK(cudaMemcpy(d.ci, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
    } else {
        MRS_CUDA_OK(cudaMemcpy(d.ci, h->col_idx, (size_t)h->nnz * d.ib, cudaMemcpyHostToDevice));
    }
    MRS_CUDA_OK(cudaMemcpy(d.v, h->values, (size_t)h->nnz * d.vb, cudaMemcpyHostToDevice));
    for (int64_t i = 0; i < h->nrows; ++i)
        d.max_row = std::max<int>(d.max_row, (int)(rp[i + 1] - rp[i]));
    // rows far longer than the mean (AMG coarse operators): whole-CTA path
    if (h->nrows > 0 && h->nnz > 0) {
        const int64_t mean = (h->nnz + h->nrows - 1) / h->nrows;
        const int64_t thr = std::max<int64_t>(64, 4 * mean);
        std::vector<int32_t> lr;
        for (int64_t i = 0; i < h->nrows; ++i)
            if (rp[i + 1] - rp[i] > thr) lr.push_back((int32_t)i);
        if (!lr.empty() && (int64_t)lr.size() * 8 <= h->nrows) {
            d.long_rows = dalloc<int32_t>(lr.size(), owned);
            if (!d.long_rows) return MRS_ERR_ALLOC;
            MRS_CUDA_OK(cudaMemcpy(d.long_rows, lr.data(), lr.size() * 4, cudaMemcpyHostToDevice));
            d.n_long = (int)lr.size();
            d.long_thr = (int)thr;
        }
    }
    if (h->slab_base) {
        if (h->idx_bytes != 2 || h->slab_shift < 0 || h->slab_shift > 30) return MRS_ERR_ARG;
        const int64_t ns = ((h->nrows - 1) >> h->slab_shift) + 1;
        d.slab_base = dalloc<int32_t>((size_t)ns, owned);
        if (!d.slab_base) return MRS_ERR_ALLOC;
        d.slab_shift = h->slab_shift;
        MRS_CUDA_OK(cudaMemcpy(d.slab_base, h->slab_base, (size_t)ns * 4, cudaMemcpyHostToDevice));
    }
    return MRS_OK;
}

// Column of entry k (row i) of a host CSR, decoding slab-relative indices.
static inline int64_t host_col(const mrs_host_csr* h, int64_t i, int64_t k) {
    int64_t c = h->idx_bytes == 4 ? ((const uint32_t*)h->col_idx)[k]
              : h->idx_bytes == 2 ? ((const uint16_t*)h->col_idx)[k]
                                  : ((const uint8_t*)h->col_idx)[k];
    if (h->slab_base) c += h->slab_base[i >> h->slab_shift];
    return c;
}

// Level schedules of both Gauss-Seidel sweep directions of a level, as row
// descriptors in schedule order (sgs.cuh, sgs_sched.h).
static int build_sgs_schedule(const mrs_host_csr* h, LevelDev& lv, std::vector<void*>& owned) {
    const int64_t n = h->nrows;
    std::vector<int32_t> dp(n, -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; ++k)
            if (host_col(h, i, k) == i) { dp[i] = (int32_t)k; break; }
    for (int64_t i = 0; i < n; ++i)
        if (dp[i] < 0) return MRS_ERR_SINGULAR;
    for (int dir = 0; dir < 2; ++dir) {
        std::vector<int32_t> order, lptr;
        sgs_levels(n, h->row_ptr, [h](int64_t i, int64_t k) { return host_col(h, i, k); }, dir,
                   order, lptr);
        const int32_t nlev = (int32_t)lptr.size() - 1;
        std::vector<int4> meta(n);
        for (int64_t q = 0; q < n; ++q) {
            const int32_t i = order[q];
            meta[q] = make_int4(i, (int)h->row_ptr[i], (int)h->row_ptr[i + 1], dp[i]);
        }
        lv.sgs_meta[dir] = dalloc<int4>(n, owned);
        lv.sgs_lptr[dir] = dalloc<int32_t>(nlev + 1, owned);
        if (!lv.sgs_meta[dir] || !lv.sgs_lptr[dir]) return MRS_ERR_ALLOC;
        MRS_CUDA_OK(cudaMemcpy(lv.sgs_meta[dir], meta.data(), n * sizeof(int4),
                               cudaMemcpyHostToDevice));
        MRS_CUDA_OK(cudaMemcpy(lv.sgs_lptr[dir], lptr.data(), (nlev + 1) * 4,
                               cudaMemcpyHostToDevice));
        lv.sgs_nlev[dir] = nlev;
    }
    lv.sgs = true;
    return MRS_OK;
}

// Per-operator SpMM variant (kernels.cu spmm_tune), measured once at
// finalize on the plan's own level buffers: every operator the solve
// multiplies with (A_l, R_l, P_l) gets the variant that ran fastest for it
// at the plan's m.  Scratch contents are overwritten later anyway.
void tune_operators(mrs_plan* p) {
    // measured per-operator choice only on request (knob plan_autotune): an
    // isolated cold launch mispredicts the operator inside a solve (A/B: C2
    // 2.43 -> 2.50 ms with it, profiles/r02_spmm_variants.txt); plans keep the
    // shape heuristic, plugin calls (a product on its own) are measured
    if (!spmm_autotune_enabled() || !plan_autotune()) return;
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
    const int64_t m = p->m;
    auto zero = [&](double* buf, int64_t rows, bool f32) {
        if (buf) cudaMemsetAsync(buf, 0, (f32 ? 4 : 8) * (size_t)rows * m, s);
    };
    const bool mg = p->desc.precond == MRS_PC_MG;
    // cold-cache conditions: an L2-sized read between tuning launches (the
    // solve streams far more than L2 between two uses of one operator)
    const int64_t fn = (160ll << 20) / 8;
    double* flush = nullptr;
    if (cudaMalloc(&flush, fn * 8) != cudaSuccess) { cudaGetLastError(); flush = nullptr; }
    else cudaMemsetAsync(flush, 0, fn * 8, s);
    const int64_t fl = flush ? fn : 0;
    for (size_t l = 0; l < p->L.size(); ++l) {
        LevelDev& lv = p->L[l];
        if (l > 0 && !mg) break;
        double* x = (l == 0 || !mg) ? p->p : lv.xa;
        double* y = (l == 0 || !mg) ? p->q : lv.r;
        const bool f = lv.f32;
        zero(x, lv.vrows, f);
        if (lv.A.present() && x && y)
            lv.A.variant = spmm_tune(lv.A, x, y, m, s, nullptr, Builder::vp(f, f), flush, fl);
        if (!mg || l + 1 >= p->L.size()) continue;
        LevelDev& lc = p->L[l + 1];
        if (lv.R.present() && lv.r && lc.b) {
            zero(lv.r, lv.vrows, f);
            lv.R.variant = spmm_tune(lv.R, lv.r, lc.b, m, s, nullptr, Builder::vp(f, lc.f32),
                                     flush, fl);
        }
        if (lv.P.present() && lc.xa && lv.r) {
            zero(lc.xa, lc.vrows, lc.f32);
            lv.P.variant = spmm_tune(lv.P, lc.xa, lv.r, m, s, nullptr, Builder::vp(lc.f32, f),
                                     flush, fl);
        }
    }
    cudaStreamSynchronize(s);
    if (flush) cudaFree(flush);
    cudaStreamDestroy(s);
    cudaGetLastError();
}

// diagonal of a host CSR in full precision (core.py:500-510); MRS_ERR_SINGULAR
// when a row has no structural diagonal or a zero diagonal entry.
int host_diag(const mrs_host_csr* h, std::vector<double>& d) {
    d.assign(h->nrows, 0.0);
    for (int64_t i = 0; i < h->nrows; ++i) {
        bool found = false;
        for (int64_t k = h->row_ptr[i]; k < h->row_ptr[i + 1]; ++k) {
            int64_t c = h->idx_bytes == 4 ? ((const uint32_t*)h->col_idx)[k]
                      : h->idx_bytes == 2 ? ((const uint16_t*)h->col_idx)[k]
                                          : ((const uint8_t*)h->col_idx)[k];
            if (h->slab_base) c += h->slab_base[i >> h->slab_shift];
            if (c == i) {
                d[i] = h->val_bytes == 8 ? ((const double*)h->values)[k]
                                         : (double)((const float*)h->values)[k];
                found = true;
                break;
            }
        }
        if (!found) return MRS_ERR_SINGULAR;
    }
    return MRS_OK;
}

}  // namespace

extern "C" {

int mrs_plan_create(const mrs_plan_desc* desc, mrs_plan** out) {
    if (!desc || !out) return MRS_ERR_ARG;
    if (desc->m < 1 || desc->m > kMaxM || desc->nrows < 1) return MRS_ERR_ARG;
    if (desc->method < MRS_METHOD_CG || desc->method > MRS_METHOD_DIRECT) return MRS_ERR_UNSUPPORTED;
    if (desc->precond < MRS_PC_NONE || desc->precond > MRS_PC_CHEB) return MRS_ERR_UNSUPPORTED;
    if (desc->method == MRS_METHOD_STATIONARY &&
        !(desc->precond == MRS_PC_JACOBI || desc->precond == MRS_PC_SGS || desc->precond == MRS_PC_MG))
        return MRS_ERR_UNSUPPORTED;
    if (desc->method == MRS_METHOD_DIRECT && desc->precond != MRS_PC_NONE) return MRS_ERR_UNSUPPORTED;
    if (desc->precond == MRS_PC_CHEB && desc->pre.order < 1) return MRS_ERR_ARG;
    for (const mrs_smoother* sm : {&desc->pre, &desc->post})
        if (desc->precond == MRS_PC_MG &&
            (sm->kind < MRS_SMOOTH_JACOBI || sm->kind > MRS_SMOOTH_SGS ||
             (sm->kind == MRS_SMOOTH_SGS && (sm->direction < 0 || sm->direction > 2))))
            return MRS_ERR_UNSUPPORTED;
    if (desc->precond == MRS_PC_SGS && (desc->pc_direction < 0 || desc->pc_direction > 2))
        return MRS_ERR_UNSUPPORTED;
    int nl = desc->precond == MRS_PC_MG ? desc->nlevels : 1;
    if (nl < 1) return MRS_ERR_ARG;
    mrs_plan* p = new mrs_plan();
    p->desc = *desc;
    p->n = desc->nrows;
    p->m = desc->m;
    p->L.resize(nl);
    *out = p;
    return MRS_OK;
}

int mrs_plan_set_level(mrs_plan* p, int32_t l, const mrs_host_csr* A, const mrs_host_csr* P,
                       const mrs_host_csr* R, double lmin, double lmax) {
    if (!p || l < 0 || l >= (int)p->L.size() || !A) return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    LevelDev& lv = p->L[l];
    int rc;
    if ((rc = upload_csr(A, lv.A, p->owned))) return rc;
    if ((rc = upload_csr(P, lv.P, p->owned))) return rc;
    if ((rc = upload_csr(R, lv.R, p->owned))) return rc;
    lv.lmin = lmin; lv.lmax = lmax;
    std::vector<double> d;
    // smoothers / Jacobi need the diagonal; the coarsest MG level and a plain
    // Krylov solve do not (the reference only checks it where it divides)
    const bool need_diag = p->desc.precond != MRS_PC_NONE &&
                           !(l == (int)p->L.size() - 1 && p->desc.precond == MRS_PC_MG);
    if (need_diag) {
        if ((rc = host_diag(A, d))) return rc;
        for (double v : d)
            if (v == 0.0) return MRS_ERR_SINGULAR;
        lv.d = dalloc<double>(d.size(), p->owned);
        if (!lv.d) return MRS_ERR_ALLOC;
        MRS_CUDA_OK(cudaMemcpy(lv.d, d.data(), d.size() * 8, cudaMemcpyHostToDevice));
    }
    const mrs_plan_desc& ds = p->desc;
    const bool sgs_level = (ds.precond == MRS_PC_SGS && l == 0) ||
                           (ds.precond == MRS_PC_MG && need_diag &&
                            (ds.pre.kind == MRS_SMOOTH_SGS || ds.post.kind == MRS_SMOOTH_SGS));
    if (sgs_level && (rc = build_sgs_schedule(A, lv, p->owned))) return rc;
    return MRS_OK;
}

int mrs_plan_set_coarse_inverse(mrs_plan* p, const double* inv, int64_t nc) {
    if (!p || !inv || nc < 1) return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    p->inv = dalloc<double>((size_t)nc * nc, p->owned);
    if (!p->inv) return MRS_ERR_ALLOC;
    p->nc = nc;
    MRS_CUDA_OK(cudaMemcpy(p->inv, inv, (size_t)nc * nc * 8, cudaMemcpyHostToDevice));
    return MRS_OK;
}

int mrs_plan_set_dense_tail(mrs_plan* p, int32_t l, const double* op, int64_t n) {
    if (!p || !op || n < 1) return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    if (p->desc.precond != MRS_PC_MG || l < 1 || l >= (int)p->L.size() - 1) return MRS_ERR_ARG;
    if (!p->L[l].A.present() || p->L[l].A.nrows != n) return MRS_ERR_ARG;
    p->tail_op = dalloc<double>((size_t)n * n, p->owned);
    if (!p->tail_op) return MRS_ERR_ALLOC;
    p->tail_n = n;
    p->dense_from = l;
    MRS_CUDA_OK(cudaMemcpy(p->tail_op, op, (size_t)n * n * 8, cudaMemcpyHostToDevice));
    return MRS_OK;
}

int mrs_plan_finalize(mrs_plan* p, void* stream) {
    (void)stream;
    if (!p) return MRS_ERR_ARG;
    if (p->finalized) return MRS_OK;
    const int64_t n = p->n, m = p->m;
    auto& o = p->owned;
    if (!p->L[0].A.present() || p->L[0].A.nrows != n) return MRS_ERR_STATE;
    // layout: rows owned, halo landing offsets, allocated vector rows
    for (size_t l = 0; l < p->L.size(); ++l) {
        LevelDev& lv = p->L[l];
        lv.nloc = lv.A.nrows;
        lv.hA.recv_row0 = lv.nloc;
        lv.hR.recv_row0 = lv.nloc;
    }
    for (size_t l = 0; l < p->L.size(); ++l) {
        LevelDev& lv = p->L[l];
        if (l + 1 < p->L.size()) lv.hP.recv_row0 = p->L[l + 1].nloc;
        int64_t halo = std::max(lv.hA.nrecv, lv.hR.nrecv);
        if (l > 0) halo = std::max<int64_t>(halo, p->L[l - 1].hP.nrecv);
        lv.vrows = lv.nloc + halo;
        if (lv.replicated && lv.slice_rows && p->comm)
            lv.vrows = std::max<int64_t>(lv.vrows, (int64_t)p->comm->nranks * lv.slice_rows);
        for (Halo* h : {&lv.hA, &lv.hR, &lv.hP})
            if (h->nsend) {
                h->sendbuf = dalloc<double>((size_t)h->nsend * m, o);
                if (!h->sendbuf) return MRS_ERR_ALLOC;
            }
        lv.A.halo = &lv.hA;
        lv.R.halo = &lv.hR;
        lv.P.halo = &lv.hP;
    }
    if (p->desc.precond == MRS_PC_MG) {
        for (size_t l = 0; l + 1 < p->L.size(); ++l) {
            LevelDev& lv = p->L[l];
            if (!lv.A.present() || !lv.P.present() || !lv.R.present()) return MRS_ERR_STATE;
        }
        if (!p->inv || p->nc != p->L.back().A.nrows) return MRS_ERR_STATE;
        if (p->desc.vec32) {
            // fp32 V-cycle vectors: levels 1 .. (collapsed tail or coarsest) - 1,
            // single GPU, Jacobi / Chebyshev smoothing (the Gauss-Seidel sweep
            // and the dense kernels stay double)
            const mrs_plan_desc& d = p->desc;
            // (PBiCGStab's pipelined recurrences need a linear preconditioner:
            // float rounding inside M makes them drift past its instability check)
            if (p->dist || d.pre.kind == MRS_SMOOTH_SGS || d.post.kind == MRS_SMOOTH_SGS ||
                d.method == MRS_METHOD_PBICGSTAB)
                return MRS_ERR_UNSUPPORTED;
            if (p->m > 32 || (p->m & (p->m - 1)) != 0) return MRS_ERR_UNSUPPORTED;
            const int end = p->dense_from >= 1 ? p->dense_from : (int)p->L.size() - 1;
            for (int l = 1; l < end; ++l) p->L[l].f32 = true;
            if (d.vec32 == 2) {
                // level 0 too: the "fp32 preconditioner" (Krylov vectors stay double);
                // MultiGrid as the SOLVER iterates on the double X itself
                if (d.method == MRS_METHOD_STATIONARY || end < 1) return MRS_ERR_UNSUPPORTED;
                p->L[0].f32 = true;
            }
        }
        for (size_t l = 0; l < p->L.size(); ++l) {
            LevelDev& lv = p->L[l];
            // float levels: the same element count in half the bytes
            const int64_t nl = lv.f32 ? (lv.vrows + 1) / 2 : lv.vrows;
            if (l > 0 || lv.f32) lv.b = dalloc<double>(nl * m, o);
            lv.xa = dalloc<double>(nl * m, o);
            lv.xb = dalloc<double>(nl * m, o);
            lv.r = dalloc<double>(nl * m, o);
            const mrs_plan_desc& d = p->desc;
            bool cheb = d.pre.kind == MRS_SMOOTH_CHEBYSHEV || d.post.kind == MRS_SMOOTH_CHEBYSHEV;
            if (cheb && l + 1 < p->L.size()) {
                lv.dva = dalloc<double>(nl * m, o);
                lv.dvb = dalloc<double>(nl * m, o);
                if (!(lv.lmin > 0.0 && lv.lmin < lv.lmax)) return MRS_ERR_ARG;
            }
            if (!lv.xa || !lv.xb || !lv.r || ((l > 0 || lv.f32) && !lv.b)) return MRS_ERR_ALLOC;
        }
    } else if (p->desc.precond == MRS_PC_JACOBI || p->desc.precond == MRS_PC_SGS) {
        if (!p->L[0].d) return MRS_ERR_STATE;
    } else if (p->desc.precond == MRS_PC_CHEB) {
        LevelDev& lv = p->L[0];
        if (!lv.d) return MRS_ERR_STATE;
        if (!(lv.lmin > 0.0 && lv.lmin < lv.lmax)) return MRS_ERR_ARG;
        const int64_t nl = lv.vrows;
        lv.r = dalloc<double>(nl * m, o);
        lv.dva = dalloc<double>(nl * m, o);
        lv.dvb = dalloc<double>(nl * m, o);
        if (!lv.r || !lv.dva || !lv.dvb) return MRS_ERR_ALLOC;
    }
    if (p->desc.method == MRS_METHOD_DIRECT && (!p->inv || p->nc != n)) return MRS_ERR_STATE;
    for (const LevelDev& lv : p->L)
        if (lv.sgs && p->dist) return MRS_ERR_UNSUPPORTED;   // one-leaf sweep order only
    size_t V = (size_t)p->L[0].vrows * m;   // level-0 Krylov vectors carry the A0 halo
    double** vecs[] = {&p->B, &p->X, &p->r, &p->r0, &p->p, &p->q, &p->v, &p->s,
                       &p->t, &p->ph, &p->sh, &p->z, &p->zt};
    for (double** v : vecs) {
        *v = dalloc<double>(V, o);
        if (!*v) return MRS_ERR_ALLOC;
    }
    p->own_B = p->B;
    p->own_X = p->X;
    if (p->desc.method == MRS_METHOD_PBICGSTAB) {
        double** pv[] = {&p->rinit, &p->zacc, &p->w, &p->yv, &p->chk, &p->pa, &p->pb};
        for (double** v : pv) {
            *v = dalloc<double>(V, o);
            if (!*v) return MRS_ERR_ALLOC;
        }
    }
    p->st = dalloc<SolveState>(1, o);
    p->history = dalloc<double>((size_t)(p->desc.max_iters + 1) * m, o);
    p->partials = dalloc<double>((size_t)max_grid() * kMaxK * m, o);
    p->ticket = dalloc<unsigned int>(1, o);
    p->red_out = dalloc<double>(kMaxK * m, o);
    if (!p->st || !p->history || !p->partials || !p->ticket || !p->red_out) return MRS_ERR_ALLOC;
    MRS_CUDA_OK(cudaMemset(p->ticket, 0, sizeof(unsigned int)));
    SolveState hs;
    memset(&hs, 0, sizeof(hs));
    hs.tol = p->desc.rel_tol;
    hs.m = (int)m;
    hs.max_iters = p->desc.max_iters;
    hs.history = p->history;
    hs.err_col = 1 << 30;
    hs.merged = p->desc.merged ? 1 : 0;
    hs.drift_limit = p->desc.drift_limit > 0.0 ? p->desc.drift_limit : 1e3;
    hs.nodrift = 1;
    for (int c = 0; c < kMaxM; ++c) { hs.one[c] = 1.0; hs.neg_one[c] = -1.0; }
    MRS_CUDA_OK(cudaMemcpy(p->st, &hs, sizeof(hs), cudaMemcpyHostToDevice));
    p->overlap = (int)halo_overlap();
    if (p->dist) {
        MRS_CUDA_OK(cudaStreamCreateWithFlags(&p->cstream, cudaStreamNonBlocking));
        MRS_CUDA_OK(cudaEventCreateWithFlags(&p->ev_pack, cudaEventDisableTiming));
        MRS_CUDA_OK(cudaEventCreateWithFlags(&p->ev_comm, cudaEventDisableTiming));
    }
    MRS_CUDA_OK(cudaMallocHost(&p->st_host, sizeof(SolveState)));
    MRS_CUDA_OK(cudaMallocHost(&p->hist_host, sizeof(double) * (size_t)(p->desc.max_iters + 1) * m));
    MRS_CUDA_OK(cudaEventCreate(&p->ev0));
    MRS_CUDA_OK(cudaEventCreate(&p->ev1));
    tune_operators(p);
    p->finalized = true;
    // estimate the per-iteration byte model / kernel count once
    Program pg;
    build_program(p, true, pg);
    p->it_bytes = pg.body_bytes;
    p->body_kernels = (int)pg.body.size();
    p->fixed_kernels = (int)(pg.pro.size() + pg.epi.size()) + 1;
    return MRS_OK;
}

int mrs_plan_solve(mrs_plan* p, const double* B, double* X, int32_t x_is_zero,
                   int32_t host_buffers, void* stream, mrs_stats* stats, double* final_rel,
                   double* history) {
    if (!p || !B || !X) return MRS_ERR_ARG;
    if (!p->finalized) return MRS_ERR_STATE;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)p->n * p->m * 8;
    cudaMemcpyKind in = host_buffers ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    cudaMemcpyKind outk = host_buffers ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const int gi = x_is_zero ? 1 : 0;
    // device buffers of a single-GPU plan are bound into the graph in place:
    // no staging copies of B and X (distributed plans need the halo rows of
    // their own level-0 vectors, host buffers need the copies anyway)
    const bool bind = p->desc.exec == 0 && !host_buffers && !p->dist &&
                      p->L[0].vrows == p->n && ((uintptr_t)B & 15u) == 0 &&
                      ((uintptr_t)X & 15u) == 0 && (const double*)B != X;
    const double* gB = bind ? B : p->own_B;
    double* gX = bind ? X : p->own_X;
    if (!bind) {
        MRS_CUDA_OK(cudaMemcpyAsync(p->own_B, B, bytes, in, s));
        if (!x_is_zero) MRS_CUDA_OK(cudaMemcpyAsync(p->own_X, X, bytes, in, s));
    }
    if (x_is_zero) MRS_CUDA_OK(cudaMemsetAsync(gX, 0, bytes, s));
    MRS_CUDA_OK(cudaEventRecord(p->ev0, s));
    cudaGraphExec_t gexec = nullptr;
    if (p->desc.exec == 0) {
        for (auto& bg : p->graphs)
            if (bg.gi == gi && bg.B == gB && bg.X == gX) gexec = bg.e;
        if (!gexec) {
            if (p->graphs.size() >= 8) {         // bounded cache: drop the oldest binding
                auto it = p->graphs.begin();
                while (it != p->graphs.end() && it->B == p->own_B) ++it;
                if (it != p->graphs.end()) {
                    cudaGraphExecDestroy(it->e);
                    cudaGraphDestroy(it->g);
                    p->graphs.erase(it);
                }
            }
            p->B = const_cast<double*>(gB);
            p->X = gX;
            cudaGraph_t g = nullptr;
            const int rc = capture_graph(p, x_is_zero != 0, s, &g, &gexec);
            p->B = p->own_B;
            p->X = p->own_X;
            if (rc != MRS_OK) {
                // e.g. collectives that cannot live inside a conditional body:
                // fall back to one captured body graph per iteration
                cudaGetLastError();
                p->desc.exec = 2;
                gexec = nullptr;
                if (bind) {        // staged path from here on
                    MRS_CUDA_OK(cudaMemcpyAsync(p->own_B, B, bytes, in, s));
                    MRS_CUDA_OK(cudaMemcpyAsync(p->own_X, X, bytes, in, s));
                }
            } else {
                p->graphs.push_back({gi, gB, gX, g, gexec});
            }
        }
    }
    if (p->desc.exec == 0) {
        MRS_CUDA_OK(cudaGraphLaunch(gexec, s));
    } else if (p->desc.exec == 2) {
        if (!p->body_exec[gi]) {
            Program pg;
            build_program(p, x_is_zero != 0, pg);
            p->pro_list[gi] = pg.pro;
            p->epi_list[gi] = pg.epi;
            cudaStream_t cs;
            MRS_CUDA_OK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            MRS_CUDA_OK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
            cudaError_t e = cudaSuccess;
            for (int u = 0; u < kDistUnroll && e == cudaSuccess; ++u) {
                gate_kernel<<<1, 1, 0, cs>>>(p->st);
                e = cudaGetLastError();
                if (e == cudaSuccess) e = run_list(pg.body, cs);
            }
            cudaGraph_t g = nullptr;
            cudaError_t e2 = cudaStreamEndCapture(cs, &g);
            cudaStreamDestroy(cs);
            if (e != cudaSuccess || e2 != cudaSuccess) return MRS_ERR_CUDA;
            MRS_CUDA_OK(cudaGraphInstantiate(&p->body_exec[gi], g, 0));
            p->body_graph[gi] = g;
        }
        if (!p->stop_host) MRS_CUDA_OK(cudaMallocHost(&p->stop_host, sizeof(int)));
        set_cond_kernel<<<1, 1, 0, s>>>(p->st, 0, 0);
        MRS_CUDA_OK(cudaGetLastError());
        MRS_CUDA_OK(run_list(p->pro_list[gi], s));
        for (;;) {
            MRS_CUDA_OK(cudaMemcpyAsync(p->stop_host, &p->st->stop, sizeof(int),
                                        cudaMemcpyDeviceToHost, s));
            MRS_CUDA_OK(cudaStreamSynchronize(s));
            if (*p->stop_host) break;
            MRS_CUDA_OK(cudaGraphLaunch(p->body_exec[gi], s));
        }
        MRS_CUDA_OK(run_list(p->epi_list[gi], s));
    } else {
        Program pg;
        // eager: no conditional handle; the host polls st->stop per iteration
        set_cond_kernel<<<1, 1, 0, s>>>(p->st, 0, 0);
        MRS_CUDA_OK(cudaGetLastError());
        build_program(p, x_is_zero != 0, pg);
        MRS_CUDA_OK(run_list(pg.pro, s));
        for (;;) {
            int stop = 0;
            MRS_CUDA_OK(cudaMemcpyAsync(&stop, &p->st->stop, sizeof(int), cudaMemcpyDeviceToHost, s));
            MRS_CUDA_OK(cudaStreamSynchronize(s));
            if (stop) break;
            MRS_CUDA_OK(run_list(pg.body, s));
        }
        MRS_CUDA_OK(run_list(pg.epi, s));
    }
    MRS_CUDA_OK(cudaEventRecord(p->ev1, s));
    if (!(bind && p->desc.exec == 0)) MRS_CUDA_OK(cudaMemcpyAsync(X, p->X, bytes, outk, s));
    const size_t hbytes = sizeof(double) * (size_t)(p->desc.max_iters + 1) * p->m;
    MRS_CUDA_OK(cudaMemcpyAsync(p->st_host, p->st, sizeof(SolveState), cudaMemcpyDeviceToHost, s));
    if (history)
        MRS_CUDA_OK(cudaMemcpyAsync(p->hist_host, p->history, hbytes, cudaMemcpyDeviceToHost, s));
    MRS_CUDA_OK(cudaStreamSynchronize(s));
    const SolveState& hs = *p->st_host;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p->ev0, p->ev1);
    if (stats) {
        stats->iterations = hs.it;
        stats->status = hs.err;
        stats->breakdown_column = hs.err == MRS_OK ? -1 : hs.err_col;
        stats->breakdown_site = hs.err_site;
        stats->device_ms = ms;
    }
    if (final_rel) memcpy(final_rel, hs.final_rel, sizeof(double) * p->m);
    if (history) memcpy(history, p->hist_host, sizeof(double) * (size_t)(hs.it + 1) * p->m);
    return hs.err;
}

int mrs_plan_set_comm(mrs_plan* p, mrs_comm* c) {
    if (!p || !c) return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    p->comm = c;
    p->dist = true;     // also with one rank: exercises the split-reduction path
    return MRS_OK;
}

int mrs_plan_set_layout(mrs_plan* p, int32_t l, int32_t replicated, int64_t slice_row0,
                        int64_t slice_rows) {
    if (!p || l < 0 || l >= (int)p->L.size()) return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    LevelDev& lv = p->L[l];
    lv.replicated = replicated != 0;
    lv.slice_row0 = slice_row0;
    lv.slice_rows = slice_rows;
    return MRS_OK;
}

int mrs_plan_set_halo(mrs_plan* p, int32_t l, int32_t which, int64_t nsend, const int32_t* send_idx,
                      const int32_t* send_counts, const int32_t* recv_counts) {
    if (!p || !p->comm || l < 0 || l >= (int)p->L.size() || which < 0 || which > 2)
        return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    LevelDev& lv = p->L[l];
    Halo& h = which == 0 ? lv.hA : (which == 1 ? lv.hR : lv.hP);
    const int R = p->comm->nranks;
    h.scount.assign(send_counts, send_counts + R);
    h.rcount.assign(recv_counts, recv_counts + R);
    h.sdisp.assign(R, 0);
    h.rdisp.assign(R, 0);
    int64_t ns = 0, nr = 0;
    for (int q = 0; q < R; ++q) {
        h.sdisp[q] = (int)ns; ns += h.scount[q];
        h.rdisp[q] = (int)nr; nr += h.rcount[q];
    }
    if (ns != nsend) return MRS_ERR_ARG;
    h.nsend = (int)ns;
    h.nrecv = (int)nr;
    if (ns) {
        h.send_idx = dalloc<int32_t>((size_t)ns, p->owned);
        if (!h.send_idx) return MRS_ERR_ALLOC;
        MRS_CUDA_OK(cudaMemcpy(h.send_idx, send_idx, (size_t)ns * 4, cudaMemcpyHostToDevice));
    }
    return MRS_OK;
}

int mrs_plan_set_interior(mrs_plan* p, int32_t l, int32_t which, int64_t ilo, int64_t ihi) {
    if (!p || !p->comm || l < 0 || l >= (int)p->L.size() || which < 0 || which > 2 || ilo < 0 ||
        ihi < ilo)
        return MRS_ERR_ARG;
    if (p->finalized) return MRS_ERR_STATE;
    LevelDev& lv = p->L[l];
    Halo& h = which == 0 ? lv.hA : (which == 1 ? lv.hR : lv.hP);
    h.ilo = ilo;
    h.ihi = ihi;
    return MRS_OK;
}

double mrs_plan_iteration_bytes(const mrs_plan* p) { return p ? p->it_bytes : 0.0; }

// Warm per-launch timing of one iteration body: after `iters` eager
// iterations (warm caches, realistic data), each launch of the body is
// captured R times back-to-back into its own graph and timed with CUDA
// events; us[i] = device time per launch (no host launch gaps).
int mrs_plan_profile(mrs_plan* p, const double* B, int32_t iters, void* stream, double* us,
                     int32_t cap,
                     int32_t* count) {
    if (!p || !p->finalized || !us || !count || iters < 1) return MRS_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    Program pg;
    build_program(p, true, pg);
    const size_t bytes = (size_t)p->n * p->m * 8;
    if (B) MRS_CUDA_OK(cudaMemcpyAsync(p->B, B, bytes, cudaMemcpyDeviceToDevice, s));
    MRS_CUDA_OK(cudaMemsetAsync(p->X, 0, bytes, s));
    set_cond_kernel<<<1, 1, 0, s>>>(p->st, 0, 0);
    MRS_CUDA_OK(run_list(pg.pro, s));
    for (int it = 0; it < iters; ++it) MRS_CUDA_OK(run_list(pg.body, s));
    MRS_CUDA_OK(cudaStreamSynchronize(s));
    const int n = (int)pg.body.size();
    const int R = 20;
    cudaEvent_t e0, e1;
    MRS_CUDA_OK(cudaEventCreate(&e0));
    MRS_CUDA_OK(cudaEventCreate(&e1));
    cudaStream_t cs;
    MRS_CUDA_OK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    *count = n;
    for (int i = 0; i < n && i < cap; ++i) {
        cudaGraph_t g;
        MRS_CUDA_OK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
        for (int r = 0; r < R; ++r) pg.body[i](cs);
        MRS_CUDA_OK(cudaStreamEndCapture(cs, &g));
        cudaGraphExec_t ge;
        MRS_CUDA_OK(cudaGraphInstantiate(&ge, g, 0));
        MRS_CUDA_OK(cudaGraphLaunch(ge, s));
        MRS_CUDA_OK(cudaEventRecord(e0, s));
        MRS_CUDA_OK(cudaGraphLaunch(ge, s));
        MRS_CUDA_OK(cudaEventRecord(e1, s));
        MRS_CUDA_OK(cudaStreamSynchronize(s));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        us[i] = 1e3 * ms / R;
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    cudaStreamDestroy(cs);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return MRS_OK;
}
// Name of the (first) kernel body launch `idx` runs, for profiles: the launch
// is captured into a scratch graph (not executed) and its kernel node read.
int mrs_plan_launch_name(mrs_plan* p, int32_t idx, char* buf, int32_t len) {
    if (!p || !p->finalized || !buf || len < 2) return MRS_ERR_ARG;
    Program pg;
    build_program(p, true, pg);
    if (idx < 0 || idx >= (int)pg.body.size()) return MRS_ERR_ARG;
    cudaStream_t cs;
    MRS_CUDA_OK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    MRS_CUDA_OK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    cudaError_t e = pg.body[idx](cs);
    cudaError_t e2 = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess || e2 != cudaSuccess) return MRS_ERR_CUDA;
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    std::string name = "(no kernel)";
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp;
        const char* nm = nullptr;
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess &&
            cudaFuncGetName(&nm, kp.func) == cudaSuccess && nm)
            name = nm;
        break;
    }
    cudaGraphDestroy(g);
    cudaGetLastError();
    snprintf(buf, (size_t)len, "%s", name.c_str());
    return MRS_OK;
}

int mrs_plan_kernel_count(const mrs_plan* p) { return p ? p->body_kernels : 0; }
int mrs_plan_fixed_kernel_count(const mrs_plan* p) { return p ? p->fixed_kernels : 0; }

void mrs_plan_destroy(mrs_plan* p) { delete p; }

}  // extern "C"
