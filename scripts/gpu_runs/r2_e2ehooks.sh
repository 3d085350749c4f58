mkdir -p gpurun_out/e2eh
for m in resnet50 densenet201; do python scripts/e2e_hooks.py $m >> gpurun_out/e2eh/out.txt 2>&1; done
cat gpurun_out/e2eh/out.txt
