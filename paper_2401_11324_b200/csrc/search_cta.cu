// Instances of search_cta_kernel (bang_search_cta.cuh): one CTA per query,
// per-query distance table in shared memory, 16-byte code rows.
#include "bang_search_cta.cuh"
#include "bang_pick.h"

namespace bang {

template <int NT, int SUB, int MV>
static const void *cta_kernel_ptr(bool hdr) {
    return hdr ? reinterpret_cast<const void *>(&search_cta_kernel<NT, SUB, MV, true>)
               : reinterpret_cast<const void *>(&search_cta_kernel<NT, SUB, MV, false>);
}

const void *pick_cta_kernel(int nt, int sub, int mv, bool hdr) {
#define BANG_C(N, S, V) \
    if (nt == N && sub == S && mv == V) return cta_kernel_ptr<N, S, V>(hdr);
    BANG_C(64, 4, 2) BANG_C(128, 4, 2) BANG_C(256, 4, 2)
    BANG_C(64, 2, 3) BANG_C(128, 2, 3) BANG_C(256, 2, 3)
    BANG_C(64, 0, 2) BANG_C(128, 0, 2) BANG_C(256, 0, 2)
    BANG_C(64, 0, 3) BANG_C(128, 0, 3) BANG_C(256, 0, 3)
#undef BANG_C
    return nullptr;
}

}  // namespace bang
