M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:tc_block -c 2 --csv python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,3]" > gpurun_out/abl5d_new.csv 2>&1
(cd _ab_split && timeout 300 ncu --metrics $M --clock-control none -k regex:tc_block -c 2 --csv python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,3]" > ../gpurun_out/abl5d_old.csv 2>&1)
