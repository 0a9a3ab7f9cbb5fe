python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cs in 1 2 8 32 64; do
  for c in 2 4; do
    KARETO_BL_CSTRIDE=$cs timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s6_b${c}_cs${cs}.log 2>&1; echo c${c}_cs${cs}_rc=$?
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "selection or config1 or tiny or w1 or edge" > gpurun_out/s6_tests.log 2>&1; echo t_rc=$?
