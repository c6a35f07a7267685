# A/B of the fused chain + Sigma dataflow (MRA_CHSIG) on C2 / C3: per-class device times, log L must be bitwise equal
mkdir -p gpurun_out
for c in C2 C3; do
  timeout 300 python tools/run_eval.py --config $c --evals 3 --prof > gpurun_out/ab_${c}_base.log 2>&1
  for lag in 16 40 96; do
    MRA_CHSIG=1 MRA_CS_LAG=$lag timeout 300 python tools/run_eval.py --config $c --evals 3 --prof > gpurun_out/ab_${c}_cs${lag}.log 2>&1
  done
done
grep -H "eval 2\|kernel classes" gpurun_out/ab_*.log
timeout 900 python -m pytest tests/test_gpu_chsig.py -x -q > gpurun_out/chsig_test.log 2>&1; echo rc=$? >> gpurun_out/chsig_test.log
