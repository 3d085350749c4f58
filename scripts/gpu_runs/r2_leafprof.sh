set -x
mkdir -p gpurun_out/lp
python scripts/leaf_one.py 128 3 > gpurun_out/lp/leaf_one.txt 2>&1
python scripts/leaf_one.py 128 1 >> gpurun_out/lp/leaf_one.txt 2>&1
python scripts/leaf_prof.py > gpurun_out/lp/leaf_prof.txt 2>&1
cat gpurun_out/lp/*.txt
