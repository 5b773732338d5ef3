for v in base l2 base l2; do
  cp _ab/libssn_$v.so paper_2312_16733_b200/libssn.so
  if [ $v = l2 ] && [ ! -f /tmp/mbdone ]; then touch /tmp/mbdone; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-families --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], {k:v['bs64_us'] for k,v in d['per_subnet'].items()})"
done
for v in base l2; do cp _ab/libssn_$v.so paper_2312_16733_b200/libssn.so; echo $v; bash tools/mb_ncu.sh "0" "3,5,14" 2>&1 | grep dbg; done
cp _ab/libssn_l2.so paper_2312_16733_b200/libssn.so
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
