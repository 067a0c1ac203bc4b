#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) on smoke() (the C1 chain in fp32 / SIMT and a
# 3-band bf16 VGG slice) and on a full-width ResNet conv2_x slice (scripts/sanitize_case.py: fused
# bottleneck, fused pointwise dgrad + wgrad, CTA-pair kernels) -> gpurun_out/<tag>_sanitize_<tool>.txt   (1 GPU, under gpurun)
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/${TAG}_sanitize_${tool}.txt 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py \
    > gpurun_out/${TAG}_sanitize_resnet_${tool}.txt 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitize_resnet_${tool}.txt
done
