mkdir -p gpurun_out
V=paper_1712_02248_b200/build_var/drain1/libcnmf_b200.so
CNMF_XS=tf32 timeout 600 python tools/rf_accuracy.py c3 2>&1 | grep span | cut -c1-120
CNMF_XS=tf32 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_k_tf32.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_k_tf32.txt | tr '\n' ' '; echo
CNMF_LIB=$V CNMF_XS=tf32 timeout 600 python tools/rf_accuracy.py c3 2>&1 | grep span | cut -c1-120
CNMF_LIB=$V CNMF_XS=tf32 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_k_d1.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_k_d1.txt | tr '\n' ' '; echo
CNMF_LIB=$V CNMF_XS=f16 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_k_d1f16.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_k_d1f16.txt | tr '\n' ' '; echo
timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_k.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_k.json')); print('c3', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'])"
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_k4.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_k4.json')); print('c4', d['value'], d['compress_seconds'], d['hals_ms_per_iteration'])"
