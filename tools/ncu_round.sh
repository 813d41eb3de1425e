CMD="python bench.py --ncu-step --no-cpu-baseline"
$CMD > gpurun_out/r01_plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/r01_ncu1.log 2>&1
echo "ncu1 rc=$?"
$CMD > gpurun_out/r01_plain2.log 2>&1 && ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Tc1x1Dgrad -s 32 -c 3 -o gpurun_out/r01_c1dgrad $CMD > gpurun_out/r01_ncu2.log 2>&1
echo "ncu2 rc=$?"
