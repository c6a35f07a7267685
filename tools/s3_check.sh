mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gputest.log 2>&1; echo rc=$? >> gpurun_out/s3_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/s3_bench_C3.json 2> gpurun_out/s3_bench_C3.err
