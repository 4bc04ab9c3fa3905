# Round-2 measurement set on one B200 (run under gpurun; outputs in gpurun_out/):
# GPU tests, smoke, bench lines C2/C3/C4 (+ reference arm at C4), the C4 bench's
# ncu launch list, full ncu captures of the HALS kernel (C4, longest launch),
# the X-stream kernel (C4) and the fp64 range-finder contraction (C3).
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
for c in c2 c3; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_c4.json 2> gpurun_out/bench_reference_c4.err; echo "ref rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_c4_launches.csv > gpurun_out/r02_c4_launch_summary.txt 2>&1
bash tools/hals_ncu.sh c4 30 hals_c4 > gpurun_out/hals_ncu.log 2>&1; echo "hals ncu rc=$?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:xs_tc_kernel -s 2 -c 2 -o gpurun_out/xs_c4 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/xs_ncu.log 2>&1; echo "xs ncu rc=$?"
$NCU -i gpurun_out/xs_c4.ncu-rep --page details --csv > gpurun_out/xs_c4_details.csv 2>/dev/null; rm -f gpurun_out/xs_c4.ncu-rep
timeout 900 $NCU --set full --clock-control none -k regex:xs_i8_kernel -s 1 -c 2 -o gpurun_out/xs64_c3 -f python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/xs64_ncu.log 2>&1; echo "xs64 ncu rc=$?"
$NCU -i gpurun_out/xs64_c3.ncu-rep --page details --csv > gpurun_out/xs64_c3_details.csv 2>/dev/null; rm -f gpurun_out/xs64_c3.ncu-rep
timeout 900 $NCU --set full --clock-control none -k regex:xs_i8_kernel -s 1 -c 2 -o gpurun_out/xsi8_c4 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/xsi8_c4_ncu.log 2>&1; echo "xs_i8 c4 ncu rc=$?"
$NCU -i gpurun_out/xsi8_c4.ncu-rep --page details --csv > gpurun_out/xsi8_c4_details.csv 2>/dev/null; rm -f gpurun_out/xsi8_c4.ncu-rep
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c3_launches.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "c3 launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_c3_launches.csv > gpurun_out/r02_c3_launch_summary.txt 2>&1
ls -la gpurun_out; du -sh gpurun_out
