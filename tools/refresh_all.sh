# Round refresh: every bench line, the reference arm, the Mandelbrot launch
# list and one ncu --set full capture per hot kernel.
set -x
bash tools/refresh_r1.sh
bash tools/prof_all.sh
