# per-kernel pipe utilisation of one CIFAR step (bench plan: L5 HX), B = 32768
python -c "import __graft_entry__ as g; g.build()"
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -s 21 -c 7 --csv python tools/plan_time.py --batch 32768 --reps 1 --plan '{"2": [1, 0, 6]}' > gpurun_out/r2_ncu_step.csv 2> gpurun_out/r2_ncu_step.err
tail -3 gpurun_out/r2_ncu_step.err
