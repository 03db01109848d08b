set -x
mkdir -p gpurun_out
prof() {  # cfg kernel tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 \
     -o gpurun_out/prof_$3 -f python tools/prof_run.py $1 2 > gpurun_out/prof_$3.log 2>&1
  echo $3=$?
  python tools/ncu_summary.py gpurun_out/prof_$3.ncu-rep > gpurun_out/prof_$3.txt 2>&1
  python tools/ncu_lines.py gpurun_out/prof_$3.ncu-rep 60 > gpurun_out/prof_$3_lines.txt 2>&1
  rm -f gpurun_out/prof_$3.ncu-rep
}
python tools/prof_run.py 2 2 && python tools/prof_run.py 4 2 && {
prof 2 k_pairs_main c2_pairs_main
prof 2 k_pairs_mids c2_pairs_mids
prof 4 k_pairs_main c4_pairs_main
prof 4 k_c5_light c4_c5_light
prof 4 k_c5_mid c4_c5_mid
prof 4 "k_c5_heavy" c4_c5_heavy
}
