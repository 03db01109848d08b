set -x
prof() {  # cfg kernel tag [lib]
  EVOKE_LIB_PATH=$4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 \
     -o gpurun_out/prof_$3 -f python tools/prof_run.py $1 2 > gpurun_out/prof_$3.log 2>&1
  echo $3=$?
  python tools/ncu_summary.py gpurun_out/prof_$3.ncu-rep > gpurun_out/prof_$3.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof_$3.ncu-rep 60 > gpurun_out/prof_$3_lines.txt 2>&1
  rm -f gpurun_out/prof_$3.ncu-rep
}
python tools/prof_run.py 2 2 && EVOKE_LIB_PATH=tools/_ref/libevoke_ref.so python tools/prof_run.py 2 2 && {
prof 2 k_pairs_main c2new_main ""
prof 2 k_pairs_mids c2new_mids ""
prof 2 k_pairs_main c2old_main tools/_ref/libevoke_ref.so
prof 2 k_pairs_mids c2old_mids tools/_ref/libevoke_ref.so
prof 2 k_pairs_heavy c2old_heavy tools/_ref/libevoke_ref.so
}
