mkdir -p gpurun_out
timeout 900 python tools/rf_kappa.py c1 c2 c3 c4 > gpurun_out/rf_kappa.txt 2>&1; cat gpurun_out/rf_kappa.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest_r.log
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_r_$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_r_$c.json')); r=d['roofline_xstream']; print('$c', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'], r['frac'], r['tn_frac'])" || tail -5 gpurun_out/bench_r_$c.json; done
