set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect "tests/test_gpu_fullsize.py::test_fullsize_run_matches_reference[c3]" > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['compress_seconds'], d['hals_seconds'], d['hals_ms_per_iteration'])"; done
CNMF_PROFILE=1 timeout 600 python tools/hals_profile.py c4 20 > gpurun_out/prof_c4.txt 2>&1; tail -25 gpurun_out/prof_c4.txt
