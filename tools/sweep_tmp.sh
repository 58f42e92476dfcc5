python tools/vcycle_time.py 2 base
TK_CARRY=grid python tools/vcycle_time.py 2 grid
for lc in 8 12 24; do TK_CHAIN_CHUNK=$lc python tools/vcycle_time.py 2 lc$lc; TK_CARRY=grid TK_CHAIN_CHUNK=$lc python tools/vcycle_time.py 2 glc$lc; done
python - <<'PY'
import numpy as np, glob
a = np.load('/tmp/vc_base.npy')
for f in sorted(glob.glob('/tmp/vc_*.npy')):
    b = np.load(f); print(f, np.abs(a - b).max() / np.abs(a).max())
PY
