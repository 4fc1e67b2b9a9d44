# ncu --set full of one kernel (usage: bash tools/gpu_ncu.sh tag config kernel_regex [--pipeline])
tag=$1; cfg=$2; kre=$3; extra=${4:-}
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kre" -c 1 -o gpurun_out/${tag} \
  python tools/run_once.py --config $cfg --reps 1 $extra > gpurun_out/${tag}.log 2>&1
tail -3 gpurun_out/${tag}.log
