for v in base xs2 xs4; do
  if [ $v = base ]; then L=""; else L=paper_1712_02248_b200/build_var/$v/libcnmf_b200.so; fi
  CNMF_LIB=$L timeout 600 python tools/rf_kappa.py c3 2>&1 | sed "s/^/$v /"
done
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_w_c4.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_w_c4.json')); print('c4', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'])"
CNMF_PROFILE=1 timeout 600 python tools/hals_profile.py c4 20 2>&1 | grep "B sweep\|ms/iter"
