python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/final3_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/final3_b2.log 2>&1; echo b2_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final3_ref4.log 2>&1; echo ref_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final3_tests.log 2>&1; echo t_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo smoke_rc=$?
