python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --config 2 --emulate-ranks 8 --steps 3 --warmup 1 > gpurun_out/s21_emu8.log 2>&1; echo emu_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s21_emu8_launches.csv python bench.py --config 2 --emulate-ranks 8 --steps 1 --warmup 0 > gpurun_out/s21_emu8_ncu.log 2>&1; echo ncu_rc=$?
