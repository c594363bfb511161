ncu --set full --import-source on --clock-control none -k regex:lr_sweep -s 1 -c 1 -f -o /tmp/lr4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_sass_top.py /tmp/lr4.ncu-rep 25 > gpurun_out/lr4_sass.txt 2>&1
ncu -i /tmp/lr4.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -2 > gpurun_out/lr4_hdr.txt
