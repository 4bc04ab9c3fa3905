mkdir -p gpurun_out
for v in tf32 f16 simt; do CNMF_XS=$v timeout 600 python tools/rf_accuracy.py c3 > gpurun_out/rf_$v.txt 2>&1; echo "$v rc=$?"; cat gpurun_out/rf_$v.txt; done
