for cfg in "128 24 64" "128 24 400" "64 24 32" "10 4 3" "256 8 100"; do DPK_EIG_SWEEPS=4 python scripts/jac_one.py $cfg; done
for sw in 4 6; do DPK_EIG_SWEEPS=$sw timeout 400 python scripts/eig_sizes.py; done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_dpkfac.py -m gpu -q -p no:cacheprovider -k "eig" > gpurun_out/gputest_r2p.log 2>&1; echo rc=$? >> gpurun_out/gputest_r2p.log; tail -4 gpurun_out/gputest_r2p.log
