# L1/L2 data-path counters of the attention kernels (what bounds the gathers):
# usage: bash tools/gpu_l1l2.sh <tag>   -> gpurun_out/<tag>_l1l2_<config>.csv
tag=${1:-l1l2}
M=gpu__time_duration.sum,sm__cycles_elapsed.max,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts_lookup_hit.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum
for c in c2_vector c1_bert_base c3_block; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:attn_ -c 1 --csv --log-file gpurun_out/${tag}_l1l2_$c.csv \
    python tools/run_once.py --config $c --reps 1 > gpurun_out/${tag}_l1l2_$c.log 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_ -c 1 --csv --log-file gpurun_out/${tag}_l1l2_c4_threshold.csv \
    python tools/run_once.py --config c4_threshold --pairs 32 --reps 1 > gpurun_out/${tag}_l1l2_c4_threshold.log 2>&1
echo done
