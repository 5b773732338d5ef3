timeout 600 ncu --set full --import-source on --clock-control none -k regex:dw_tma -s 3 -c 1 -o gpurun_out/ncu_dw_k7 python tools/dw_bench.py 256,56,56,192,192,7,7,1 --iters 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dw_tma -s 3 -c 1 -o gpurun_out/ncu_dw_c24 python tools/dw_bench.py 256,112,112,24,24,3,3,1 --iters 1 > /dev/null 2>&1
ls gpurun_out/ncu_dw*
