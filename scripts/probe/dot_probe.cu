// dot_probe.cu -- cost of the fused dot (CTA partials -> last-CTA fold) on
// the library's SpMM kernel: q = A p with and without (p, q), C2 fine level.
// Built against the library sources (not the .so):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -o dot_probe dot_probe.cu ../../paper_2103_07329_b200/csrc/{kernels,spmm_f64,spmm_f32}.cu
#include <stdio.h>

#include <algorithm>
#include <random>
#include <vector>

#include "../../paper_2103_07329_b200/csrc/launch.cuh"

using namespace mrs;

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e = (x);                                                                  \
        if (e != cudaSuccess) { fprintf(stderr, "%d %s\n", __LINE__, cudaGetErrorString(e)); exit(1); } \
    } while (0)

template <typename T> static T* up(const std::vector<T>& h) {
    T* d;
    CK(cudaMalloc(&d, h.size() * sizeof(T) + 256));
    CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

int main() {
    const int g = 64, n = g * g * g, m = 8;
    std::vector<int32_t> rp{0};
    std::vector<uint32_t> ci;
    std::vector<double> v;
    for (int z = 0; z < g; ++z)
        for (int y = 0; y < g; ++y)
            for (int x = 0; x < g; ++x) {
                const int i = (z * g + y) * g + x;
                auto add = [&](int j, double w) { ci.push_back(j); v.push_back(w); };
                if (z) add(i - g * g, -1);
                if (y) add(i - g, -1);
                if (x) add(i - 1, -1);
                add(i, 6);
                if (x < g - 1) add(i + 1, -1);
                if (y < g - 1) add(i + g, -1);
                if (z < g - 1) add(i + g * g, -1);
                rp.push_back((int)ci.size());
            }
    std::vector<double> hp((size_t)n * m);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& t : hp) t = U(rng);
    const int NSET = 8;   // rotate copies: each launch reads cold operands
    std::vector<DevCsr> As(NSET);
    std::vector<double*> P(NSET), Q(NSET);
    for (int k = 0; k < NSET; ++k) {
        DevCsr& A = As[k];
        A.nrows = A.ncols = n; A.nnz = (int64_t)ci.size();
        A.rp = up(rp); A.ci = up(ci); A.v = up(v); A.ib = 4; A.vb = 8;
        P[k] = up(hp);
        CK(cudaMalloc(&Q[k], hp.size() * 8));
    }
    double *partials, *out;
    unsigned* ticket;
    CK(cudaMalloc(&partials, (size_t)num_sms() * kMaxGridPerSM * kMaxK * m * 8));
    CK(cudaMalloc(&out, kMaxK * m * 8));
    CK(cudaMalloc(&ticket, 4));
    CK(cudaMemset(ticket, 0, 4));
    for (int dot = 0; dot < 2; ++dot) {
        auto run = [&](int k) {
            SpArgs a;
            memset(&a, 0, sizeof(a));
            a.x = P[k]; a.y = Q[k]; a.mode = MRS_MODE_ASSIGN;
            if (dot) {
                a.dot = 1;
                a.red.partials = partials; a.red.ticket = ticket; a.red.out = out;
                a.red.st = nullptr; a.red.epi = EPI_NONE;
            }
            CK(launch_spmm(OP_SPMV, As[k], a, m, 0));
        };
        for (int k = 0; k < NSET; ++k) run(k);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int R = 5;
        cudaEventRecord(e0);
        for (int r = 0; r < R; ++r)
            for (int k = 0; k < NSET; ++k) run(k);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("q = A p (C2 fine, m=8, u32) %s: %.2f us per launch (back-to-back, cold operands)\n",
               dot ? "WITH fused (p,q)" : "without dot    ", ms * 1e3 / (R * NSET));
    }
    return 0;
}
