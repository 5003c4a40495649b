# ncu --set full of the kernels matching $1 in one profiled C3 frame (scripts/profile_frame.py)
mkdir -p gpurun_out
pat=$1; tag=$2
cmd="python scripts/profile_frame.py"
$cmd > gpurun_out/frame_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$pat \
    -o gpurun_out/${tag} -f $cmd > gpurun_out/ncu_${tag}.log 2>&1
echo "rc=$?"
