# ncu full capture of the one-launch network kernel (CIFAR, batch 1) with source/SASS
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:net_b1 -s 45 -c 1 \
  -o gpurun_out/r2_net_cifar python tools/net_trace.py > gpurun_out/r2_net_ncu.log 2>&1
tail -3 gpurun_out/r2_net_ncu.log
