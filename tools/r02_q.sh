mkdir -p gpurun_out
timeout 900 python tools/rf_kappa.py c1 c2 c3 c4 > gpurun_out/rf_kappa.txt 2>&1; cat gpurun_out/rf_kappa.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_q.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest_q.log
