# ncu capture of the longest hals_kernel launch of a run (launches are cut at
# redraw events): list launch durations first, then a full capture of the
# longest one.   usage: bash tools/hals_ncu.sh c4 30 outname
set -x
CFG=${1:-c4}; IT=${2:-30}; OUT=${3:-hals_$CFG}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:hals_kernel --csv \
  --log-file gpurun_out/${OUT}_launches.csv python tools/hals_profile.py $CFG $IT --noprof > /dev/null 2>&1
IDX=$(python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/${OUT}_launches.csv")) if len(r)>10 and r[0]!="ID" and r[-3].startswith("gpu__time")]
d=[float(r[-1].replace(",","")) for r in rows]
print(max(range(len(d)), key=lambda i:d[i]) if d else 0)
PY
)
echo "longest launch index $IDX"
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:hals_kernel --launch-skip $IDX -c 1 \
  -o gpurun_out/$OUT -f python tools/hals_profile.py $CFG $IT --noprof > gpurun_out/${OUT}_ncu.log 2>&1; echo "ncu rc=$?"
$NCU -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${OUT}_source.csv 2>/dev/null
$NCU -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${OUT}_source.csv 60 > gpurun_out/${OUT}_hot.txt 2>&1
gzip -f gpurun_out/${OUT}_source.csv
rm -f gpurun_out/$OUT.ncu-rep
