# ncu --set full of kernels matching $1 for each variant in $2.. (bench C3, 2 launches after 4)
mkdir -p gpurun_out
pat=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset FVV_LIB; else export FVV_LIB=$PWD/_variants/$v/libfvv.so; fi
  cmd="python bench.py --steps 3 --warmup 3 --lanes 1 --no-e2e --no-cpu-baseline"
  $cmd > gpurun_out/plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$pat -s 4 -c 2 \
      -o gpurun_out/prof_$v -f $cmd > gpurun_out/ncu_$v.log 2>&1
  echo "$v rc=$?"
done
