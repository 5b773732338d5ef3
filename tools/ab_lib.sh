# A/B two prebuilt engine libraries on one box (box-to-box variance is ~3%,
# so compare within one gpurun call):
#   cp paper_2312_16733_b200/libssn.so _ab/libssn_<name>.so   (for each variant)
#   gpurun -- 'bash tools/ab_lib.sh <a> <b> [microbench cases]'
A=${1:-base}; B=${2:-new}; CASES=${3:-3,5,14}
for v in $A $B $A $B; do
  cp _ab/libssn_$v.so paper_2312_16733_b200/libssn.so
  timeout 300 python bench.py --steps 20 --warmup 3 --no-families --no-cpu --no-slackfit 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], {k:(v['bs1_us'],v['bs8_us'],v['bs64_us'],v.get('bs256_us')) for k,v in d['per_subnet'].items()})"
done
for v in $A $B; do
  cp _ab/libssn_$v.so paper_2312_16733_b200/libssn.so
  echo $v; bash tools/mb_ncu.sh "0" "$CASES" 2>&1 | grep dbg
done
cp _ab/libssn_$B.so paper_2312_16733_b200/libssn.so
