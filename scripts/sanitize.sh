#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) on the C1 chain (fp32, SIMT) and a 2-band bf16
# VGG slice (tcgen05 kernels) -> gpurun_out/<tag>_sanitize_<tool>.txt   (1 GPU, under gpurun)
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/${TAG}_sanitize_${tool}.txt 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.txt
done
