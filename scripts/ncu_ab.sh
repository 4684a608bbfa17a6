set -e
for v in base desc; do
  PHIKS_LIB_PATH=build_exp/$v/libphiks.so python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plain_$v.log 2>&1
  PHIKS_LIB_PATH=build_exp/$v/libphiks.so ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 12 -c 3 -o gpurun_out/prof_$v python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1
done
