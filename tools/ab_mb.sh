# microbench conv cases under two SSN_TC_DEBUG values: warm-L2 ncu device time + prof (dbg|32) prints
A=${1:-0}; B=${2:-0}; C=${3:-4,5,7,32}
mkdir -p gpurun_out/abmb
for d in $A $B; do
  SSN_TC_DEBUG=$d CASES=$C timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/abmb/mb_$d.csv python tools/microbench_conv.py > gpurun_out/abmb/mb_$d.log 2>&1
  SSN_TC_DEBUG=$((d | 32)) CASES=$C timeout 120 python tools/microbench_conv.py > gpurun_out/abmb/prof_$d.log 2>&1
done
