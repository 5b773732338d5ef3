# A/B two environment settings on the family rows (OFA-MBv3 / BERT) of bench.py
A=${1:-SSN_TC_DEBUG=0}; B=${2:-SSN_TC_DEBUG=0}
for v in "$A" "$B" "$A" "$B"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-slackfit --no-parity 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); f=d['families']; print('$v', round(d['value']), {fam: {s: {b: x['us'] for b, x in f[fam][s].items() if b in ('bs64', 'bs256')} for s in ('min', 'mid', 'max')} for fam in f if isinstance(f[fam], dict)})"
done
