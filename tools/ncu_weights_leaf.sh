set -e
ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:^k_weights$" -s 18 -c 1 \
    -o gpurun_out/w14 python tools/compress_profile.py 3 1048576 4 1e-6 > gpurun_out/w14.log 2>&1
python profiles/summarize_ncu.py gpurun_out/w14.ncu-rep > gpurun_out/w14.txt
python tools/ncu_lines.py gpurun_out/w14.ncu-rep 40 >> gpurun_out/w14.txt
ncu -i gpurun_out/w14.ncu-rep --page raw --csv > gpurun_out/w14_raw.csv
