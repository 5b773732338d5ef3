# A/B two prebuilt libraries (_ab/libssn_<name>.so) on the family rows of bench.py
A=${1:-base}; B=${2:-new}
for v in $A $B $A $B; do
  cp _ab/libssn_$v.so paper_2312_16733_b200/libssn.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-slackfit --no-parity 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); f=d['families']; print('$v', round(d['value']), {fam: {s: {b: x['us'] for b, x in f[fam][s].items() if b in ('bs64', 'bs256')} for s in ('min', 'mid', 'max')} for fam in f if isinstance(f[fam], dict)})"
done
cp _ab/libssn_$B.so paper_2312_16733_b200/libssn.so
