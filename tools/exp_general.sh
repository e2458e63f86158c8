# launch list of the general-pattern unfold (sparse300, ring1000, dense48) + one ncu --set full of the
# light fill kernel at sparse300
mkdir -p gpurun_out
for w in sparse300 ring1000 dense48; do
  python tools/prof_general.py $w > /dev/null 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gen_$w.csv python tools/prof_general.py $w > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_g_light" -s 3 -c 1 -o gpurun_out/glight_full -f python tools/prof_general.py sparse300 > /dev/null 2>&1; echo ncu=$?
