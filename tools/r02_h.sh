mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streaming.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/gputest_h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_h.log
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['compress_seconds'], d['hals_seconds'], d['hals_ms_per_iteration'])"; done
CNMF_PROFILE=1 timeout 600 python tools/hals_profile.py c4 20 > gpurun_out/prof_c4.txt 2>&1; tail -20 gpurun_out/prof_c4.txt
V=paper_1712_02248_b200/build_var/drain1/libcnmf_b200.so
for v in tf32 f16; do CNMF_LIB=$V CNMF_XS=$v timeout 600 python tools/rf_accuracy.py c3 > gpurun_out/rf_d1_$v.txt 2>&1; head -3 gpurun_out/rf_d1_$v.txt; done
for v in tf32 f16; do CNMF_LIB=$V CNMF_XS=$v timeout 600 python tools/c3_gpu_variants.py c3 gpurun_out/c3_d1_$v.npz > gpurun_out/c3_d1_$v.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_d1_$v.txt | tr '\n' ' '; echo; done
for v in tf32 f16; do CNMF_LIB=$V CNMF_XS=$v timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_d1_$v.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_d1_$v.json')); print('d1 $v', d['value'], d['compress_seconds'], d['roofline_xstream']['frac'], d['roofline_xstream']['tn_frac'])"; done
