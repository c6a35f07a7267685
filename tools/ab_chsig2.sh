mkdir -p gpurun_out
for lag in 200 500 2000; do
  MRA_CHSIG=1 MRA_CS_LAG=$lag timeout 300 python tools/run_eval.py --config C3 --evals 3 --prof > gpurun_out/ab2_C3_cs${lag}.log 2>&1
done
