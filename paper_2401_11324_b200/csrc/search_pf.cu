// Instances of search_pf_kernel (bang_search_pf.cuh): search_cta_kernel with
// 1 or 2 prefetch warps working one hop ahead.
#include "bang_search_pf.cuh"
#include "bang_pick.h"

namespace bang {

template <int N, int S, int V>
static const void *pf_kernel_ptr(int pfw, bool stage) {
    if (stage) return pfw == 2 ? reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 2, true>)
                               : reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 1, true>);
    return pfw == 2 ? reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 2, false>)
                    : reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 1, false>);
}

const void *pick_pf_kernel(int nt, int sub, int mv, int pfw, bool stage) {
#define BANG_P(N, S, V) \
    if (nt == N && sub == S && mv == V) return pf_kernel_ptr<N, S, V>(pfw, stage);
    BANG_P(128, 4, 2) BANG_P(256, 4, 2)
    BANG_P(128, 2, 3) BANG_P(256, 2, 3)
    BANG_P(128, 0, 2) BANG_P(256, 0, 2)
    BANG_P(128, 0, 3) BANG_P(256, 0, 3)
#undef BANG_P
    return nullptr;
}

}  // namespace bang
