mkdir -p gpurun_out/tl
python scripts/step_timeline.py resnet50 > gpurun_out/tl/resnet50.txt 2>&1
cat gpurun_out/tl/resnet50.txt
