# round 2: bench with the timed full-recompute generation + tcgen05 tensor-pipe counter probe
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_frac.log 2>&1; tail -c 3000 gpurun_out/r2_bench_frac.log
M=gpu__time_duration.sum,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv -k regex:"gemm_skinny|attn_fused|gemm_tcgen05" --log-file gpurun_out/r2_tensor_metrics_ro.csv python tools/profile_step.py --mode ro > gpurun_out/r2_ncu_tc.log 2>&1; tail -2 gpurun_out/r2_ncu_tc.log
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv -k regex:"gemm_skinny|attn_fused|gemm_tcgen05" --log-file gpurun_out/r2_tensor_metrics_full.csv python tools/profile_step.py --mode full > gpurun_out/r2_ncu_tc2.log 2>&1; tail -2 gpurun_out/r2_ncu_tc2.log
