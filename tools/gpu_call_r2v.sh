timeout 300 ./tools/sortbench_r2 > gpurun_out/sortbench.log 2>&1; echo sb_rc=$?
