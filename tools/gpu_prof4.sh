# r02 profiles on the bench config (config 4): launch list, then ncu --set full of the top
# kernels (one report each; summaries + raw csv kept), then serial pass times of configs 3, 5
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-config 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches4.csv $B > gpurun_out/ncu_launch4.log 2>&1; echo launches=$?
python tools/launch_summary.py gpurun_out/launches4.csv 5 | head -40
for ks in ${PROF_KERNELS:-k_c5_light k_c5_mid k_c5_heavy k_pairs_main k_pairs_mids k_pairs_heavy}; do
  k=${ks%%:*}; skip=${PROF_SKIP:-3}; [ "$k" != "$ks" ] && skip=${ks#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
     -o gpurun_out/prof4_$k -f $B > gpurun_out/prof4_$k.log 2>&1
  echo $k=$?
  python tools/ncu_summary.py gpurun_out/prof4_$k.ncu-rep > gpurun_out/prof4_$k.txt 2>&1
  ncu -i gpurun_out/prof4_$k.ncu-rep --page raw --csv > gpurun_out/prof4_${k}_raw.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/prof4_$k.ncu-rep 60 > gpurun_out/prof4_${k}_lines.txt 2>&1
  rm -f gpurun_out/prof4_$k.ncu-rep
done
if [ -z "$NO_BIG" ]; then
EVOKE_DEBUG=1 timeout 600 python tools/dev_timing.py 3 2 --serial > gpurun_out/timing3.log 2>&1; echo t3=$?
tail -25 gpurun_out/timing3.log
EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py 5 1 --warm 0 --serial > gpurun_out/timing5.log 2>&1; echo t5=$?
tail -40 gpurun_out/timing5.log
fi
