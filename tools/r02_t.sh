mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streaming.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/gputest_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_t.log
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_t_$c.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_t_$c.json')); print('$c', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'])"; done
CNMF_PROFILE=1 timeout 600 python tools/hals_profile.py c4 20 > gpurun_out/prof_c4.txt 2>&1; tail -20 gpurun_out/prof_c4.txt
