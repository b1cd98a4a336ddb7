timeout -s KILL 1200 python scripts/th_table.py --out gpurun_out/th_table.csv > gpurun_out/th_table.log 2>&1
