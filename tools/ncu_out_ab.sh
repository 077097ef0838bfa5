for c in c3 c5 c2; do for v in 0 1; do
WINO_OUT_TMA=$v WINO_GEMM_VARIANT=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:output -s 3 -c 2 python bench.py --steps 2 --warmup 3 --config $c --extra "" --nets "" --no-cpu-baseline 2>/dev/null | grep -E "k_output|duration|dram__" | sed "s/^/$c tma=$v /" | cut -c1-140
done; done
