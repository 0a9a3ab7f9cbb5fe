python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"DeviceRadixSort(Onesweep|Histogram)Kernel" -c 14 -o gpurun_out/s17_sort_c4 python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/s17_ncu4.log 2>&1; echo f4_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"DeviceRadixSort(Onesweep|Histogram)Kernel" -c 14 -o gpurun_out/s17_sort_c2 python bench.py --config 2 --profile-only --steps 1 --warmup 0 > gpurun_out/s17_ncu2.log 2>&1; echo f2_rc=$?
