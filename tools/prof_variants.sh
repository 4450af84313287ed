# ncu --set full of the first launch of kernel regex $1 for each variant library
K=${1:-tangent_row}
for f in paper_2411_14315_b200/variants/*.so; do v=$(basename $f .so); HBGPU_LIB=$f timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -c ${2:-1} -o gpurun_out/prof_$v -f python bench.py --no-solve --no-cpu-baseline --spmv-reps 1 --steps 1 --warmup 3 > gpurun_out/prof_$v.log 2>&1; echo "$v rc=$?"; done
