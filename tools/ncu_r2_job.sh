set -e
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for w in c3 c2 c4-32 c4-64; do python tools/profile_step.py --workload $w > gpurun_out/plain_$w.log 2>&1; done
for w in c3 c4-32 c4-64; do ncu --metrics $M --clock-control none -k regex:"gemm_bf16|scatter|plan_scan|combine" -s 15 -c 5 --csv --log-file gpurun_out/r2_launches_$w.csv python tools/profile_step.py --workload $w > /dev/null 2>&1; done
ncu --metrics $M --clock-control none -k regex:"gemm_bf16|scatter|plan_scan|combine" -s 18 -c 6 --csv --log-file gpurun_out/r2_launches_c2.csv python tools/profile_step.py --workload c2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_tc_kernel|scatter_kernel" -s 8 -c 2 -o gpurun_out/r2_gate_dispatch python tools/profile_step.py --workload c3 > gpurun_out/ncu_full.log 2>&1
echo done
