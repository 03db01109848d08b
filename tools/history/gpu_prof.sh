# one ncu --set full capture per heavy kernel of the bench step (config 2); the text summary
# and the raw-page csv are written next to each report, and the reports themselves are
# dropped unless KEEP_REP=1 (gpurun copies back at most 64 MiB)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
# entries are NAME or NAME:SKIP (launches of NAME to skip; default PROF_SKIP or 3)
for ks in ${PROF_KERNELS:-k_pairs_main k_c5_heavy}; do
  k=${ks%%:*}; skip=${PROF_SKIP:-3}; [ "$k" != "$ks" ] && skip=${ks#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
     -o gpurun_out/prof_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_$k.log 2>&1
  echo $k=$?
  python tools/ncu_summary.py gpurun_out/prof_$k.ncu-rep > gpurun_out/prof_$k.txt 2>&1
  ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_raw.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/prof_$k.ncu-rep ${PROF_LINES:-80} > gpurun_out/prof_${k}_lines.txt 2>&1
  [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/prof_$k.ncu-rep
done
