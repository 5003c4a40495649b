# every kernel of one C3 frame: launch list + ncu --set full (executed-work counters)
mkdir -p gpurun_out
tag=${1:-r2}
cmd="env FVV_FORK=0 python scripts/profile_frame.py"  # (one chain: launch order = stage order)
$cmd > gpurun_out/frame_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_frame_launches.csv $cmd > /dev/null 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o gpurun_out/${tag}_frame_full -f $cmd > gpurun_out/ncu_frame.log 2>&1
echo "rc=$?"
