timeout 300 ncu --set full --import-source on --clock-control none -k regex:se_expand -s 20 -c 1 -o gpurun_out/se_expand python tools/prof_forward.py --family mbv3 --batch 256 --steps 1 --warmup 1 --subnets max > /dev/null 2>&1
ls -la gpurun_out/se_expand*
