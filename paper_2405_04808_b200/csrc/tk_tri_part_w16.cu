// tri_rows_part instantiations for 16 warp(s) per CTA (see tk_tri_part.cuh)
#include "tk_tri_part.cuh"

namespace tk {
template int part_dispatch_x<16, 1>(const tk_level*, int, bool, const double*, const double*, double*,
                                     double, const double*, cudaStream_t, double*, const double*, int);
}  // namespace tk
