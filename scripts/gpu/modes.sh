# the GPU parity suite under each executor mode switch
for m in "FVV_DEVICE_PLAN=0" "FVV_FRAME_GRAPH=0" "FVV_PDL=0 FVV_FORK=0"; do
  env $m python -m pytest tests -m gpu -q -x > gpurun_out/mode.log 2>&1
  echo "$m: $(tail -1 gpurun_out/mode.log)"
done
