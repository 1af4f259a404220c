# Round-1 evidence for profiles/: launch lists (gpu__time_duration.sum) of each
# bench workload and one full capture of each hot kernel.  Run under gpurun:
#   gpurun --timeout 1500 -- 'bash tools/r1_profiles.sh'
set -x
N="ncu --clock-control none"
$N --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/r1_launches_mel.csv python bench.py --steps 2 --warmup 1 --no-breakdown > /dev/null 2>&1
for w in cqt1992v2 cqt2010v2 train; do
  $N --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/r1_launches_$w.csv python bench.py --workload $w --steps 2 --warmup 1 --no-breakdown > /dev/null 2>&1
done
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o gpurun_out/r1_mel_gemm python tools/ncu_target.py mel 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o gpurun_out/r1_stft_gemm python tools/ncu_target.py stft 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:egemm_kernel -s 1 -c 1 -o gpurun_out/r1_cqt1992_egemm python tools/ncu_target.py cqt1992v2 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o gpurun_out/r1_cqt1992_sched python tools/ncu_target.py cqt1992v2 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_tc_kernel -s 1 -c 1 -o gpurun_out/r1_cqt2010 python tools/ncu_target.py cqt2010v2 2 > /dev/null 2>&1
# training step: rgemm launches per step = W@S, dW, dS+coef, dK (wide pair)
$N --set full --import-source on -k regex:rgemm_kernel -s 6 -c 1 -o gpurun_out/r1_train_coef python tools/ncu_train_target.py 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:rgemm_kernel -s 7 -c 1 -o gpurun_out/r1_train_dk python tools/ncu_train_target.py 2 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o gpurun_out/r1_train_fwd python tools/ncu_train_target.py 2 > /dev/null 2>&1
ls -la gpurun_out
