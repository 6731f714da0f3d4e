set -x
for w in mandelbrot gaussian binomial nbody ray mandelbrot_f32 mandelbrot_periodic; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench3_$w.json 2> gpurun_out/bench3_$w.err
  echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/bench3_reference.json 2> gpurun_out/bench3_reference.err
echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches3_mandelbrot.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3_launch.log 2>&1
echo "ncu rc=$?"
