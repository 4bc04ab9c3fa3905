mkdir -p gpurun_out
timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_p.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_p.txt | tr '\n' ' '; echo; grep "final\|relF" gpurun_out/c3_p.txt
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_p_$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_p_$c.json')); r=d['roofline_xstream']; print('$c', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'], r['frac'], r['tn_frac'])" || tail -5 gpurun_out/bench_p_$c.json; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_p.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest_p.log
