python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/final4_b4.log 2>&1; echo b4_rc=$?
timeout 900 python bench.py --config 2 > gpurun_out/final4_b2.log 2>&1; echo b2_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final4_ref4.log 2>&1; echo ref_rc=$?
