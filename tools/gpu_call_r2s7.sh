python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_BL_SUB=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_full or config1 or fingerprint or full_size_config2 or edge or tiny or agent" > gpurun_out/s7_tests_sub3.log 2>&1; echo t3_rc=$?
for sub in 0 2 3 5; do
  for cs in 1 2; do
    for c in 2 4; do
      KARETO_BL_SUB=$sub KARETO_BL_CSTRIDE=$cs timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s7_b${c}_sub${sub}_cs${cs}.log 2>&1; echo c${c}_sub${sub}_cs${cs}_rc=$?
    done
  done
done
