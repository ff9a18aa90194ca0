set -x
timeout 300 python scripts/expt/time_bs6.py 1 2 3 5 7 15 > gpurun_out/bs6_keep.log 2>&1
SB200_LIB=scripts/expt/_alt/libsb200.so timeout 300 python scripts/expt/time_bs6.py 1 2 3 5 7 15 >> gpurun_out/bs6_keep.log 2>&1
for L in paper_2009_10917_b200/lib/libsb200.so scripts/expt/_alt/libsb200.so; do
SB200_LIB=$L timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_bs6 -s 2 -c 1 python scripts/expt/time_bs6.py 1 2>&1 | grep -E "dram__|gpu__time" >> gpurun_out/bs6_keep.log
done
cat gpurun_out/bs6_keep.log
