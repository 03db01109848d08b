set -x
python tools/prof_run.py 4 1 > gpurun_out/p2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/p2_launches.csv python tools/prof_run.py 4 1 > gpurun_out/p2_ncu.log 2>&1
echo ncu=$?
python tools/launch_summary.py gpurun_out/p2_launches.csv > gpurun_out/p2_summary.txt 2>&1
head -50 gpurun_out/p2_summary.txt
