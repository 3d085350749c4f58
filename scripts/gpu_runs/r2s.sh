for l in 1 0; do for n in 128 64 100; do DPK_LEAF16=$l python scripts/leaf16_one.py $n 3; done; done
python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "inverse or spd or factor_inv or chol or precondition" > gpurun_out/gputest_r2s.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2s.log; tail -5 gpurun_out/gputest_r2s.log
for l in 1 0; do echo "LEAF16=$l"; SPD_ONLY=4608 DPK_LEAF16=$l python scripts/inv_factor_one.py 20; DPK_LEAF16=$l python scripts/inv_factor_one.py 20; done
