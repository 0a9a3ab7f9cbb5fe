timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_run.py trace1 > gpurun_out/san2_race_trace1.log 2>&1; echo race_rc=$?
