# round-end evidence at the current code: smoke, the whole GPU suite, the bench line, the
# config-4 launch list, ncu --set full of the top kernels (summaries + raw csv), traffic.json
# inputs, configs 3 and 5 serial pass times
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ -z "$NO_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 5000 gpurun_out/bench.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-config 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches4.csv $B > gpurun_out/ncu_launch4.log 2>&1; echo launches=$?
python tools/launch_summary.py gpurun_out/launches4.csv 9 > gpurun_out/launches4_summary.txt 2>&1; head -40 gpurun_out/launches4_summary.txt
for k in ${PROF_KERNELS:-k_c5_light k_c5_mid k_c5_heavy k_pairs_main k_pairs_mids}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
     -o gpurun_out/prof4_$k -f $B > gpurun_out/prof4_$k.log 2>&1
  echo $k=$?
  python tools/ncu_summary.py gpurun_out/prof4_$k.ncu-rep > gpurun_out/prof4_$k.txt 2>&1
  ncu -i gpurun_out/prof4_$k.ncu-rep --page raw --csv > gpurun_out/prof4_${k}_raw.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/prof4_$k.ncu-rep 60 > gpurun_out/prof4_${k}_lines.txt 2>&1
  rm -f gpurun_out/prof4_$k.ncu-rep
done
EVOKE_DEBUG=1 timeout 600 python tools/dev_timing.py 3 2 --serial > gpurun_out/timing3.log 2>&1; echo t3=$?
tail -18 gpurun_out/timing3.log
EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py 5 1 --warm 0 --serial > gpurun_out/timing5.log 2>&1; echo t5=$?
tail -18 gpurun_out/timing5.log
