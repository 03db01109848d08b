# developer: A/B of the in-tree build against variants/libevoke_$VARS.so on configs $CFGS (serial pass times)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in ${CFGS:-4 3}; do
  for v in main ${VARS}; do
    if [ $v = main ]; then L=""; else L="EVOKE_LIB_PATH=variants/libevoke_$v.so"; fi
    env $L timeout 600 python tools/dev_timing.py $c ${REPS:-3} --serial > gpurun_out/var_${c}_$v.log 2>&1; echo $c $v=$?
    grep "wall\|${GREP:-pair_pass\|cycles5}" gpurun_out/var_${c}_$v.log
  done
done
