#!/bin/bash
# Regenerates the measured evidence under profiles/ for the CURRENT library build, on one B200:
#   gpurun --timeout 3000 -- 'bash tools/refresh_evidence.sh r02'
# writes gpurun_out/ev/: bench lines of every config (never under a profiler), the ncu launch list of
# the default bench command, --set full captures of the dominant kernels (summarised per source line by
# tools/ncu_lines.py) and the DRAM traffic files bench.py reads (tools/traffic.py; tied to the library
# fingerprint).  Copy what should be judged from gpurun_out/ev/ into profiles/.
set -u
R=${1:-r02}
O=gpurun_out/ev
mkdir -p $O
NCU="ncu --clock-control none"

# 1. DRAM traffic per kernel group of this build (bench.py's roofline.traffic)
for c in cfg4 cfg2 cfg3 cfg1 cfg5; do
  python tools/traffic.py $c > $O/traffic_$c.log 2>&1 && cp profiles/traffic_$c.json $O/
done

# 2. bench lines (no profiler; they pick up this build's traffic files)
for c in cfg4 cfg2 cfg3 cfg1 cfg5; do
  python bench.py --config $c > $O/${R}_bench_$c.json 2> $O/bench_$c.err || echo "bench $c failed" >> $O/errors.log
done
python bench.py --impl reference --steps 3 --warmup 1 > $O/${R}_bench_reference_cfg4.json 2> $O/bench_ref.err

# 3. launch list of the default bench command (shares, not absolutes)
$NCU --metrics gpu__time_duration.sum -k 'regex:k_|Radix' --csv --log-file $O/${R}_ncu_launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1

# 4. full captures: the dense screen (default config), front+scan (configs[1]), transform (configs[2], configs[4])
$NCU --set full --import-source on -k regex:k_dense_screen -s 4 -c 1 -o $O/screen_cfg4 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_screen.log 2>&1
python tools/ncu_lines.py $O/screen_cfg4.ncu-rep k_dense_screen 20 > $O/${R}_ncu_full_k_dense_screen_cfg4.txt 2>&1
$NCU --set full --import-source on -k regex:k_query -s 6 -c 2 -o $O/query_cfg2 -f \
  python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_query.log 2>&1
python tools/ncu_lines.py $O/query_cfg2.ncu-rep k_query 25 > $O/${R}_ncu_full_k_query_front_scan_cfg2.txt 2>&1
$NCU --set full --import-source on -k regex:k_transform -c 1 -o $O/transform_cfg3 -f \
  python tools/transform_probe.py cfg3 10000000 1 > $O/ncu_transform3.log 2>&1
python tools/ncu_lines.py $O/transform_cfg3.ncu-rep k_transform 20 > $O/${R}_ncu_full_k_transform_cfg3.txt 2>&1
$NCU --set full --import-source on -k regex:k_transform -c 1 -o $O/transform_cfg5 -f \
  python tools/transform_probe.py cfg5 5000000 1 > $O/ncu_transform5.log 2>&1
python tools/ncu_lines.py $O/transform_cfg5.ncu-rep k_transform 20 > $O/${R}_ncu_full_k_transform_cfg5.txt 2>&1
# the reports themselves stay on the box (gpurun_out/ is capped at 64 MiB); the summaries travel
rm -f $O/screen_cfg4.ncu-rep $O/query_cfg2.ncu-rep $O/transform_cfg5.ncu-rep
ls -la $O
