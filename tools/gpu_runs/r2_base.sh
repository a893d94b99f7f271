set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_gputest.log
timeout 900 python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo rc=$?
tail -3 gpurun_out/r2_bench2.err
