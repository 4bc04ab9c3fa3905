set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:hals_kernel -c 1 -o gpurun_out/hals_c4 -f python tools/hals_profile.py c4 3 --noprof > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_c4.log
$NCU -i gpurun_out/hals_c4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/hals_c4_source.csv 2>/dev/null
$NCU -i gpurun_out/hals_c4.ncu-rep --page details --csv > gpurun_out/hals_c4_details.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/hals_c4_source.csv 50 > gpurun_out/hals_c4_hot.txt 2>&1
ls -la gpurun_out/
gzip -f gpurun_out/hals_c4_source.csv
du -sh gpurun_out
