mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest_s.log
for c in c2 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_s_$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_s_$c.json')); r=d['roofline_xstream']; print('$c', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'], r['frac'], r['tn_frac'])" || tail -5 gpurun_out/bench_s_$c.json; done
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_inv --csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e 2>/dev/null | grep chol_inv | head -3
