# developer: serial pass times of config $CFG under each env setting in $KNOBS (";"-separated)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
IFS=';'
i=0
for kv in $KNOBS; do
  i=$((i+1))
  env $kv timeout 600 python tools/dev_timing.py ${CFG:-4} ${REPS:-3} --serial > gpurun_out/knob_$i.log 2>&1; echo "[$kv]=$?"
  grep "wall\|${GREP:-cycles5}" gpurun_out/knob_$i.log
done
