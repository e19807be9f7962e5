set -x
python scripts/attn_shapes.py c2 > gpurun_out/r2_attn_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attention_tcgen05_2sm_pp --launch-count 1 -o gpurun_out/r2_attn_pp python scripts/attn_shapes.py c2 > gpurun_out/r2_ncu_attn.log 2>&1
ncu -i gpurun_out/r2_attn_pp.ncu-rep --page raw --csv > gpurun_out/r2_attn_pp_raw.csv 2>&1
ncu -i gpurun_out/r2_attn_pp.ncu-rep --page source --csv > gpurun_out/r2_attn_pp_source.csv 2>&1
ncu -i gpurun_out/r2_attn_pp.ncu-rep --page details --csv > gpurun_out/r2_attn_pp_details.csv 2>&1
ls -la gpurun_out
