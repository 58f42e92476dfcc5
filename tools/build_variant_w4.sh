#!/bin/bash
# variant of libtempokkt_b200.so with extra -D flags for the W = 4 row kernels only
# (tk_tri_part_w4.cu: n_u = 512): tools/build_variant_w4.sh <name> <flags...>
exec "$(dirname "$0")/build_variant_file.sh" tk_tri_part_w4.cu "$@"
