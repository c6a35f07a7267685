# final round-2 lines on HEAD: C0-C2, C4 bench lines and the C3 launch list (ncu, per-launch times / DRAM / DMMA)
mkdir -p gpurun_out
for c in C0 C1 C2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/f6_bench_$c.json 2> gpurun_out/f6_bench_$c.err; done
timeout 600 python bench.py --config C4 --steps 2 --warmup 3 > gpurun_out/f6_bench_C4.json 2> gpurun_out/f6_bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/f6_launches_C3.csv python tools/run_eval.py --config C3 --evals 1 > gpurun_out/f6_ncu_list.log 2>&1
echo done
