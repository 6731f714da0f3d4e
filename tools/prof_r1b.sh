# ncu --set full captures of the packed Binomial and NBody kernels (each only
# after the same command exited 0 without ncu).
set -x
python tools/profile_run.py --workload binomial > gpurun_out/plain_binomial2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:binomial_warp -s 1 -c 1 -o gpurun_out/ncu_binomial2 python tools/profile_run.py --workload binomial > gpurun_out/ncu_binomial2.log 2>&1
echo "binomial ncu rc=$?"
python tools/profile_run.py --workload nbody --steps-override 1 > gpurun_out/plain_nbody2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nbody_step -s 1 -c 1 -o gpurun_out/ncu_nbody2 python tools/profile_run.py --workload nbody --steps-override 1 > gpurun_out/ncu_nbody2.log 2>&1
echo "nbody ncu rc=$?"
