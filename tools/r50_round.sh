# R50 loop: gpu tests (engine + headline + ops), per-family timing, bench line
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python tools/profile_family.py --family r50 --batches 1,64,256 > gpurun_out/r50_family.log 2>&1; cat gpurun_out/r50_family.log | cut -c1-150
timeout 300 python tools/profile_family.py --family bert --batches 64 > gpurun_out/bert_family.log 2>&1; cat gpurun_out/bert_family.log | cut -c1-150
