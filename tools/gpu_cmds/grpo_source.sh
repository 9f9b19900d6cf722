set -x
mkdir -p gpurun_out/gsrc
python tools/prof_grpo_fused.py > gpurun_out/gsrc/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_grpo_fused" -s 1 -c 1 -o gpurun_out/gsrc/gf -f python tools/prof_grpo_fused.py > gpurun_out/gsrc/ncu.log 2>&1
ncu -i gpurun_out/gsrc/gf.ncu-rep --page source --csv --print-source sass > gpurun_out/gsrc/gf_sass.csv 2>/dev/null
ncu -i gpurun_out/gsrc/gf.ncu-rep --page raw --csv > gpurun_out/gsrc/gf_raw.csv 2>/dev/null
rm -f gpurun_out/gsrc/gf.ncu-rep
ls -la gpurun_out/gsrc
