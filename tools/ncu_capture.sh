# ncu --set full of the comparison kernel for a bench.py workload (one launch of
# the regular CTA-pair grid after warm-up) + the extra L2/SMEM metrics we track.
# usage: bash tools/ncu_capture.sh <tag> [bench.py args...]
tag=$1; shift
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    --metrics l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed_pipe_uniform.sum \
    -k regex:tensor_kernel --launch-skip ${SKIP:-4} -c 1 -f -o gpurun_out/$tag \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --verify none "$@" > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep 30 > gpurun_out/$tag.summary.txt 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
