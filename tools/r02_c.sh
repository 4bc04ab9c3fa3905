set -x
mkdir -p gpurun_out
for v in tf32 simt f16; do CNMF_XS=$v timeout 600 python tools/c3_gpu_variants.py c3 gpurun_out/c3_$v.npz > gpurun_out/c3_$v.txt 2>&1; echo "$v rc=$?"; done
python - <<'PY'
import numpy as np
r={v:np.load(f"gpurun_out/c3_{v}.npz") for v in ("tf32","simt","f16")}
for a in r:
  for b in r:
    if a<b: print(a,b,"max rel traj diff", np.max(np.abs(r[a]["err"]-r[b]["err"])/r[b]["err"]))
PY
cat gpurun_out/c3_tf32.txt
