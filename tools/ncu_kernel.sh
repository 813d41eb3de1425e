# usage: bash tools/ncu_kernel.sh <regex> <skip> <count> <out-name>
# Plain run of the one-step bench, then a --set full capture of matching launches.
CMD="python bench.py --ncu-step --no-cpu-baseline"
$CMD > gpurun_out/$4_plain.log 2>&1 && ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$1 -s $2 -c $3 -o gpurun_out/$4 $CMD > gpurun_out/$4_ncu.log 2>&1
echo "ncu rc=$?"
