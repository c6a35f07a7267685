set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f1_gputest.log 2>&1; echo rc=$? >> gpurun_out/f1_gputest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/f1_bench_C3.json 2> gpurun_out/f1_bench_C3.err
for c in C0 C1 C2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/f1_bench_$c.json 2> gpurun_out/f1_bench_$c.err; done
timeout 600 python bench.py --config C4 --steps 2 --warmup 3 > gpurun_out/f1_bench_C4.json 2> gpurun_out/f1_bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/f1_launches_C3.csv python tools/run_eval.py --config C3 --evals 1 > gpurun_out/f1_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wide_mtile -c 1 -f -o gpurun_out/f1_mtile python tools/run_eval.py --config C3 --evals 1 > gpurun_out/f1_ncu_mtile.log 2>&1
