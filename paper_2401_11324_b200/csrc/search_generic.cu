// Instances of search_kernel (bang_kernels.cuh): one warp per query, every
// ADC data flow (exact, HBM table, shared codebook, per-warp smem table).
#include "bang_kernels.cuh"
#include "bang_pick.h"

namespace bang {

template <int NPL, int SUB, int MV>
static const void *kernel_ptr() {
    return reinterpret_cast<const void *>(&search_kernel<NPL, SUB, MV>);
}

const void *pick_kernel(int npl, int sub, int mv) {
#define BANG_K(N, S, V) \
    if (npl == N && sub == S && mv == V) return kernel_ptr<N, S, V>();
    BANG_K(1, 0, 0) BANG_K(2, 0, 0) BANG_K(4, 0, 0)
    BANG_K(1, 4, 2) BANG_K(2, 4, 2) BANG_K(4, 4, 2)
    BANG_K(1, 2, 3) BANG_K(2, 2, 3) BANG_K(4, 2, 3)
    BANG_K(1, 0, 2) BANG_K(2, 0, 2) BANG_K(4, 0, 2)
    BANG_K(1, 0, 3) BANG_K(2, 0, 3) BANG_K(4, 0, 3)
#undef BANG_K
    return nullptr;
}

}  // namespace bang
