python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_run.py all > gpurun_out/s30_memcheck.log 2>&1; echo mem_rc=$?
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_run.py all > gpurun_out/s30_synccheck.log 2>&1; echo sync_rc=$?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py trace1 > gpurun_out/s30_race_trace1.log 2>&1; echo race1_rc=$?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py replay > gpurun_out/s30_race_replay.log 2>&1; echo race2_rc=$?
