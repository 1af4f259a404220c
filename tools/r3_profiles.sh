# Round-2 (late) evidence for profiles/: the new CQT2010v2 route (front / chain / conv)
# launch list and full captures, plus a bench sweep of every workload.  Run under gpurun:
#   gpurun --timeout 2400 -- 'bash tools/r3_profiles.sh'
set -x
N="ncu --clock-control none"
O=gpurun_out
$N --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r3_launches_cqt2010v2.csv python bench.py --workload cqt2010v2 --steps 2 --warmup 1 --no-breakdown --cpu-seconds 0.1 > /dev/null 2>&1
for k in front chain conv_kernel; do
  $N --set full --import-source on -k regex:cqt2010_$k -s 1 -c 1 -o $O/r3_cqt2010_$k python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
done
for w in mel melpow2 stft cqt1992v2 cqt2010v2; do
  python bench.py --workload $w > $O/r3_bench_$w.json 2> $O/r3_bench_$w.err
done
for pr in fp32 tf32; do
  python bench.py --workload mel --precision $pr --no-breakdown > $O/r3_bench_mel_$pr.json 2>&1
  python bench.py --workload train --precision $pr --no-breakdown > $O/r3_bench_train_$pr.json 2>&1
done
python bench.py --workload cqt2010v2 --precision fp32 --no-breakdown > $O/r3_bench_cqt2010v2_fp32.json 2>&1
python bench.py --impl reference --workload cqt2010v2 --steps 2 --warmup 1 > $O/r3_bench_ref_cqt2010v2.json 2>&1
ls -la $O | grep r3_
