python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_K1_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_tma.log 2>&1; echo t_rc=$?
KARETO_K1_TMA=1 timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/b4_tma.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/b4_notma.log 2>&1; echo b4n_rc=$?
KARETO_K1_TMA=1 timeout 900 python bench.py --config 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b2_tma.log 2>&1; echo b2_rc=$?
