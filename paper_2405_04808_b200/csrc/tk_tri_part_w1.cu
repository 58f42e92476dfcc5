// tri_rows_part instantiations for 1 warp(s) per CTA (see tk_tri_part.cuh)
#include "tk_tri_part.cuh"

namespace tk {
template int part_dispatch_x<1, 1>(const tk_level*, int, bool, const double*, const double*, double*,
                                     double, const double*, cudaStream_t, double*, const double*, int);
template int part_dispatch_r<1, 1>(const tk_level*, bool, const double*, const double*, double*,
                                     double, const double*, cudaStream_t);
}  // namespace tk
