// sgs_sched.h -- host-side level schedule of a sequential Gauss-Seidel
// half-sweep (see sgs.cuh for why it reproduces the sequential order).
#pragma once

#include <stdint.h>

#include <algorithm>
#include <vector>

namespace mrs {

// Forward (dir 0): row i must follow every row j < i it reads (it needs j's
// new value) and every row r < i that reads i (r needs i's old value);
// level(i) = 1 + the largest such level.  Backward (dir 1): the mirror image
// over descending rows.  `col(i, k)` = column of entry k of row i.  Output:
// rows grouped by level, ascending inside a level; lptr[nlev + 1].
template <class Col>
void sgs_levels(int64_t n, const int64_t* rp, Col col, int dir, std::vector<int32_t>& order,
                std::vector<int32_t>& lptr) {
    std::vector<int32_t> lev(n), dep(n, -1);
    int32_t nlev = 0;
    for (int64_t t = 0; t < n; ++t) {
        const int64_t i = dir == 0 ? t : n - 1 - t;
        int32_t L = dep[i];
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t c = col(i, k);
            if (dir == 0 ? c < i : c > i) L = std::max(L, lev[c]);
        }
        lev[i] = L + 1;
        nlev = std::max(nlev, lev[i] + 1);
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t c = col(i, k);
            if (dir == 0 ? c > i : c < i) dep[c] = std::max(dep[c], lev[i]);
        }
    }
    lptr.assign(nlev + 1, 0);
    for (int64_t i = 0; i < n; ++i) lptr[lev[i] + 1]++;
    for (int32_t q = 0; q < nlev; ++q) lptr[q + 1] += lptr[q];
    std::vector<int32_t> fill(lptr.begin(), lptr.end() - 1);
    order.resize(n);
    for (int64_t i = 0; i < n; ++i) order[fill[lev[i]]++] = (int32_t)i;
}

}  // namespace mrs
