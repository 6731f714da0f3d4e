set -x
export ECL_NO_STREAMED_INPUTS=1
cap() {
  python tools/profile_run.py --workload $1 $3 > gpurun_out/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/ncu_$1 \
      python tools/profile_run.py --workload $1 $3 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
}
cap gaussian gaussian_tiled
cap binomial binomial_warp
cap ray ray_persistent
