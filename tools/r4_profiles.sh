# Late round-2 evidence: the CQT2010v2 route after the back-end merge (front + back), launch list
# and full captures, and the bench line.  gpurun --timeout 1800 -- 'bash tools/r4_profiles.sh'
set -x
N="ncu --clock-control none"
O=gpurun_out
$N --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r4_launches_cqt2010v2.csv python bench.py --workload cqt2010v2 --steps 2 --warmup 1 --no-breakdown --cpu-seconds 0.1 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_front -s 1 -c 1 -o $O/r4_cqt2010_front python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_back -s 0 -c 1 -o $O/r4_cqt2010_back python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
python bench.py --workload cqt2010v2 > $O/r4_bench_cqt2010v2.json 2> $O/r4_bench_cqt2010v2.err
python tools/dbg_front_prof.py > $O/r4_front_prof.txt 2>&1
python tools/dbg_back_prof.py > $O/r4_back_prof.txt 2>&1
ls -la $O | grep r4_
