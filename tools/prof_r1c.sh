set -x
python tools/profile_run.py --workload gaussian > gpurun_out/plain_gaussian3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gaussian_tiled -s 1 -c 1 -o gpurun_out/ncu_gaussian3 python tools/profile_run.py --workload gaussian > gpurun_out/ncu_gaussian3.log 2>&1
echo "gaussian ncu rc=$?"
python tools/profile_run.py --workload ray > gpurun_out/plain_ray3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ray_persistent -s 1 -c 1 -o gpurun_out/ncu_ray3 python tools/profile_run.py --workload ray > gpurun_out/ncu_ray3.log 2>&1
echo "ray ncu rc=$?"
