# warm per-kernel times (frame_gaps) of experiment builds: kvariants.sh PATTERN v1 v2 ...
pat=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset FVV_LIB; else export FVV_LIB=$PWD/_variants/$v/libfvv.so; fi
  echo "== $v"; python scripts/frame_gaps.py --frames 10 2>/dev/null | grep -E "busy|$pat"
done
