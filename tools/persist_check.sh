#!/bin/bash
# configs[3]/[1] V-cycle + solve with and without the L2-persisting Arnoldi w
for p in 1 0; do
  echo "TK_ARNOLDI_PERSIST=$p"
  TK_ARNOLDI_PERSIST=$p timeout 600 python tools/run_configs.py 3 1 --solve 2>/dev/null
done
