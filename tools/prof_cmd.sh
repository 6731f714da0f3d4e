set -x
./tools/probe/hostbw > gpurun_out/hostbw.txt 2>&1
for w in gaussian binomial ray; do
  python tools/profile_run.py --workload $w > gpurun_out/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"gaussian_tiled|binomial_warp|ray_persistent" -s 1 -c 1 -o gpurun_out/ncu_$w python tools/profile_run.py --workload $w > gpurun_out/ncu_$w.log 2>&1
  echo "$w ncu rc=$?"
done
python tools/profile_run.py --workload nbody --steps-override 1 > gpurun_out/plain_nbody.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nbody_step -s 1 -c 1 -o gpurun_out/ncu_nbody python tools/profile_run.py --workload nbody --steps-override 1 > gpurun_out/ncu_nbody.log 2>&1
echo "nbody ncu rc=$?"
python tools/profile_run.py --workload mandelbrot > gpurun_out/plain_mandel.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_mandel.csv python tools/profile_run.py --workload mandelbrot > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
