export PYTHONDONTWRITEBYTECODE=1
for i in 1 2; do
for lib in paper_2502_00021_b200/libpxr.so build/var/libpxr_640.so build/var/libpxr_704.so; do
  for m in "Humanoid video" "HalfCheetah none" "Walker2d video" "Ant color"; do
    set -- $m
    echo -n "$(basename $lib) "
    PXR_LIB_PATH=$PWD/$lib timeout 120 python tools/prof_step.py --timed 50 --model "$1" --mode "$2" | tail -1
  done
done; done
