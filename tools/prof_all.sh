# ncu --set full capture of one launch of every hot kernel (each after the
# same command ran clean without ncu); summaries -> profiles/<round>/.
set -x
export ECL_NO_STREAMED_INPUTS=1  # whole-package launches, as in the timed resident runs
cap() {  # workload kernel-regex extra-args [launches-to-skip]
  python tools/profile_run.py --workload $1 $3 > gpurun_out/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-1} -c 1 -o gpurun_out/ncu_$1 \
      python tools/profile_run.py --workload $1 $3 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
}
cap mandelbrot mandel_persistent
cap gaussian gaussian_sep
cap binomial binomial_hw
cap nbody nbody_step "--steps-override 1"
cap ray ray_persistent "" 44  # a heavy 1M-pixel piece (mid-image), not a sky piece
cap mandelbrot_f32 mandel_x2
