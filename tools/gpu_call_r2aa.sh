python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san2_memcheck.log 2>&1; echo mem_rc=$?
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/san2_synccheck.log 2>&1; echo sync_rc=$?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py trace > gpurun_out/san2_race_trace.log 2>&1; echo race_t_rc=$?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py replay > gpurun_out/san2_race_replay.log 2>&1; echo race_r_rc=$?
