python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
KARETO_DEBUG=1 timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --e2e-steps 0 --cpu-full 0 > gpurun_out/s11_b3.log 2>&1; echo b3_rc=$?
KARETO_DEBUG=1 timeout 2400 python tools/config3_fullsize_sample.py --per-cell 12 > gpurun_out/s11_c3full.log 2>&1; echo c3full_rc=$?
