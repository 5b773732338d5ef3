# A/B two environment settings with one library on one box (box-to-box variance
# is ~3%, so compare within one gpurun call):
#   gpurun -- 'bash tools/ab_env.sh "SSN_X=0" "SSN_X=1" [pytest-targets]'
# (a bare number is taken as an SSN_TC_DEBUG value)
A=${1:-SSN_TC_DEBUG=0}; B=${2:-SSN_TC_DEBUG=0}; T=${3:-}
case $A in *=*) ;; *) A="SSN_TC_DEBUG=$A";; esac
case $B in *=*) ;; *) B="SSN_TC_DEBUG=$B";; esac
mkdir -p gpurun_out/ab
if [ -n "$T" ]; then timeout 900 python -m pytest -x -q $T > gpurun_out/ab/pytest.log 2>&1; tail -3 gpurun_out/ab/pytest.log; fi
for v in "$A" "$B" "$A" "$B"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-families --no-cpu --no-slackfit 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['e2e']['value']), {k:(v['bs1_us'], v['bs8_us'], v['bs64_us']) for k,v in d['per_subnet'].items()})"
done
