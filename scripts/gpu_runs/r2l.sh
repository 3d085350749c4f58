python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "inverse or spd or factor_inv or chol" > gpurun_out/gputest_r2l.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2l.log; tail -5 gpurun_out/gputest_r2l.log
for rl in 0 2048; do
  echo "DPK_SPD_RL=$rl"
  SPD_ONLY=4608 DPK_SPD_RL=$rl timeout 120 python scripts/inv_factor_one.py 20
  SPD_ONLY=2304 DPK_SPD_RL=$rl timeout 120 python scripts/inv_factor_one.py 20
  DPK_SPD_RL=$rl timeout 120 python scripts/inv_factor_one.py 20
done
for cap in 64 96 116 132; do echo "cap $cap"; SPD_ONLY=4608 DPK_RL_CAP=$cap timeout 120 python scripts/inv_factor_one.py 20; done
