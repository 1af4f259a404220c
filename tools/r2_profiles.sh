# Round-2 evidence for profiles/: launch lists (gpu__time_duration.sum) of each
# bench workload and one full capture of each hot kernel.  Run under gpurun:
#   gpurun --timeout 1800 -- 'bash tools/r2_profiles.sh'
set -x
N="ncu --clock-control none"
O=gpurun_out
$N --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r2_launches_mel.csv python bench.py --steps 2 --warmup 1 --no-breakdown --cpu-seconds 0.1 > /dev/null 2>&1
for w in stft cqt1992v2 cqt2010v2; do
  $N --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r2_launches_$w.csv python bench.py --workload $w --steps 2 --warmup 1 --no-breakdown --cpu-seconds 0.1 > /dev/null 2>&1
done
$N --metrics gpu__time_duration.sum -c 400 --csv --log-file $O/r2_launches_train.csv python bench.py --workload train --precision tf32 --steps 2 --warmup 1 --no-breakdown --cpu-seconds 0.1 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r2_mel_f16_gemm python tools/ncu_target.py mel 2 f16 > /dev/null 2>&1
$N --set full --import-source on -k regex:stage_rows_f16 -s 1 -c 1 -o $O/r2_stage_f16 python tools/ncu_target.py mel 2 f16 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r2_mel_tf32_gemm python tools/ncu_target.py mel 2 tf32 > /dev/null 2>&1
$N --set full --import-source on -k regex:egemm_kernel -s 1 -c 1 -o $O/r2_cqt1992_egemm python tools/ncu_target.py cqt1992v2 2 tf32 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r2_cqt1992_sched python tools/ncu_target.py cqt1992v2 2 tf32 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_tc_kernel -s 1 -c 1 -o $O/r2_cqt2010 python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r2_train_fwd python tools/ncu_train_target.py 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:rgemm_kernel -s 7 -c 1 -o $O/r2_train_dk python tools/ncu_train_target.py 2 > /dev/null 2>&1
ls -la $O | grep r2_
