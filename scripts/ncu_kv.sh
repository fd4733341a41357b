M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum
for o in 0 1; do
GESR_PROJ_ORDER=$o timeout 600 ncu --metrics $M --clock-control none --kernel-name regex:proj_kernel -c 2 --csv python scripts/kbench.py --iters 1 --out-dtype bf16 > gpurun_out/ncu_kv_o$o.csv 2>&1
done
