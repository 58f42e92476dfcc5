cd $GRAFT_REPO_ROOT
for v in default c2m4 c2m2; do
  if [ $v = default ]; then L=paper_2405_04808_b200/libtempokkt_b200.so; else L=paper_2405_04808_b200/lib_$v.so; fi
  TK_LIB_PATH=$L timeout 300 python tools/time_jacobi.py 2 $v 2>&1 | tail -1
done
python - <<'PY'
import numpy as np
a=np.load('/tmp/jac_default.npy')
for v in ['c2m4','c2m2']:
    b=np.load(f'/tmp/jac_{v}.npy'); print(v, np.abs(a-b).max()/np.abs(a).max())
PY
timeout 900 python tools/run_configs.py 0 1 3 4 --solve > gpurun_out/cfg_graph.jsonl 2>gpurun_out/cfg_graph.err; echo cfg rc=$?
cat gpurun_out/cfg_graph.jsonl
