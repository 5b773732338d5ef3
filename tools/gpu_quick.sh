# quick GPU loop: gpu tests, conv microbench, bench line, launch-list summary
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 120 python tools/microbench_conv.py 2>&1 | grep dbg | awk '{print $2, $(NF-10), $(NF-9)}'
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_new.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_new.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline_detail']['whole_net_roofline_frac'], {k:v['bs64_us'] for k,v in d['per_subnet'].items()}, {f:{k:v[k]['us'] for k in ('min','mid','max')} for f,v in d.get('families',{}).items()})" || tail -5 gpurun_out/bench_new.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_new.csv python tools/prof_forward.py --steps 1 --warmup 1 > /dev/null 2>&1; python tools/launches.py gpurun_out/launch_new.csv | head -8
