# depthwise microbench + op parity + one ncu --set full capture per bound
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k dw 2>&1 | tail -2
python tools/dw_bench.py 256,56,56,96,192,7,3,1 256,56,56,192,192,7,7,1 256,112,112,24,24,3,3,1 256,112,112,72,144,7,3,2 256,14,14,288,576,7,3,1 256,7,7,1152,1152,7,7,1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dw_tma -s 3 -c 1 -o gpurun_out/ncu_dw_k3 python tools/dw_bench.py 256,56,56,96,192,7,3,1 --iters 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dw_tma -s 3 -c 1 -o gpurun_out/ncu_dw_k7 python tools/dw_bench.py 256,56,56,192,192,7,7,1 --iters 1 > /dev/null 2>&1
