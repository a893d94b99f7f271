python -c "import __graft_entry__ as g; g.build()"
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/net_debug.py > gpurun_out/san_race.log 2>&1; tail -30 gpurun_out/san_race.log
timeout 600 compute-sanitizer --tool initcheck python tools/net_debug.py > gpurun_out/san_init.log 2>&1; grep -m5 -A12 "Uninitialized" gpurun_out/san_init.log; tail -5 gpurun_out/san_init.log
