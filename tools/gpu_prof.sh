# one ncu --set full capture per heavy kernel of the bench step (config 2)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in ${PROF_KERNELS:-k_hublocal k_pairs_shared k_pairs_global k_cycles5}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${PROF_SKIP:-3} -c 1 \
     -o gpurun_out/prof_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_$k.log 2>&1
  echo $k=$?
done
