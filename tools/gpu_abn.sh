# interleaved timing of several libpxr builds over the four BASELINE
# workloads: bash tools/gpu_abn.sh <lib> <lib> ...
export PYTHONDONTWRITEBYTECODE=1
libs=("$@")
for i in 1 2; do
  for lib in "${libs[@]}"; do
    for m in "Humanoid video" "HalfCheetah none" "Walker2d video" "Ant color"; do
      read -r model mode <<< "$m"
      echo -n "$(basename "$lib") "
      PXR_LIB_PATH=$PWD/$lib timeout 120 python tools/prof_step.py --timed 50 --model "$model" --mode "$mode" | tail -1
    done
  done
done
