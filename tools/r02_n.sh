mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f16.py -x -q -p no:cacheprovider > gpurun_out/gputest_n.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest_n.log
timeout 600 python tools/rf_accuracy.py c3 2>&1 | cut -c1-150
timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_n.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_n.txt | tr '\n' ' '; echo; grep final gpurun_out/c3_n.txt
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_n_$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_n_$c.json')); r=d['roofline_xstream']; print('$c', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'], r['frac'], r['tn_frac'])"; done
