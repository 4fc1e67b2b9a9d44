#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   bench lines for every BASELINE config (with the bounded cpu_baseline)
#   and the reference arm (C2), the per-launch kernel list of each config
#   (ncu gpu__time_duration, cold, serialised), and one `ncu --set full`
#   capture of each config's dominant kernel.
#   Usage: bash tools/evidence.sh <tag>   (outputs in gpurun_out/)
set -u
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
for c in c2_vector c3_block c4_threshold c1_bert_base c0_smoke; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $out/${tag}_bench_$c.json 2> $out/${tag}_bench_$c.err
done
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_bench_reference_c2.json 2> $out/${tag}_bench_reference.err
for c in c2_vector c3_block c4_threshold c1_bert_base c0_smoke; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-adjacent > $out/${tag}_ncu_launch_$c.log 2>&1
done
declare -A dom=([c2_vector]=colvec_kernel [c3_block]=attn_block [c4_threshold]=threshold_tc [c1_bert_base]=topk_rowsel [c0_smoke]=project)
for c in c2_vector c3_block c4_threshold c1_bert_base c0_smoke; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:${dom[$c]} -c 1 -o $out/${tag}_full_$c \
    python tools/run_once.py --config $c --reps 1 > $out/${tag}_ncu_full_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_band -c 1 -o $out/${tag}_full_c2_attn \
    python tools/run_once.py --config c2_vector --reps 1 > $out/${tag}_ncu_full_c2_attn.log 2>&1
echo done
