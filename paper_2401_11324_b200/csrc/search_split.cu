// Instances of search_split_kernel (bang_search_split.cuh): row warps build
// the next hop's keys while list warps merge the previous hop's.
#include "bang_pick.h"
#include "bang_search_split.cuh"

namespace bang {

const void *pick_split_kernel(int pl, int sub, int mv) {
#define BANG_P(L, S, V) \
    if (pl == L && sub == S && mv == V) return reinterpret_cast<const void *>(&search_split_kernel<L, S, V>);
    BANG_P(1, 4, 2) BANG_P(2, 4, 2)
    BANG_P(1, 2, 3) BANG_P(2, 2, 3)
    BANG_P(1, 0, 2) BANG_P(2, 0, 2)
    BANG_P(1, 0, 3) BANG_P(2, 0, 3)
#undef BANG_P
    return nullptr;
}

}  // namespace bang
