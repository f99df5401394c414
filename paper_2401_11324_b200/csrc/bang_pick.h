// bang_pick.h -- kernel-instance selectors.  Each search kernel family is
// instantiated in its own translation unit (search_*.cu) so nvcc compiles
// them in parallel; bang_abi.cu launches through these pointers.
#pragma once

namespace bang {
// search_kernel<NPL, SUB, MV> (search_generic.cu)
const void *pick_kernel(int npl, int sub, int mv);
// search_cta_kernel<NT, SUB, MV, HDR> (search_cta.cu)
const void *pick_cta_kernel(int nt, int sub, int mv, bool hdr);
// search_split_kernel<PL, SUB, MV> (search_split.cu), PL = neighbour slots per row thread
const void *pick_split_kernel(int pl, int sub, int mv);
}  // namespace bang
