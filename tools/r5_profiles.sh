# Round-2 late evidence: FP32 mode (3xF16 kernel gradient, staged split-mode epilogues) and the
# CQT2010v2 route after the front changes.  gpurun --timeout 2400 -- 'bash tools/r5_profiles.sh'
set -x
N="ncu --clock-control none"
O=gpurun_out
B="--no-breakdown --cpu-seconds 0.1"
$N --metrics gpu__time_duration.sum -c 200 --csv --log-file $O/r5_launches_train_fp32.csv python bench.py --workload train --precision fp32 --steps 1 --warmup 1 $B > /dev/null 2>&1
$N --metrics gpu__time_duration.sum -c 200 --csv --log-file $O/r5_launches_train_tf32.csv python bench.py --workload train --precision tf32 --steps 1 --warmup 1 $B > /dev/null 2>&1
$N --metrics gpu__time_duration.sum -c 200 --csv --log-file $O/r5_launches_mel_fp32.csv python bench.py --workload mel --precision fp32 --steps 2 --warmup 1 $B > /dev/null 2>&1
$N --metrics gpu__time_duration.sum -c 200 --csv --log-file $O/r5_launches_cqt2010v2.csv python bench.py --workload cqt2010v2 --steps 2 --warmup 1 $B > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r5_train_fp32_fwd python tools/ncu_train_target.py 2 split fp32 > /dev/null 2>&1
$N --set full --import-source on --kernel-name-base demangled -k "regex:rgemm_kernel.*\(bool\)0, \(bool\)1>" -s 1 -c 1 -o $O/r5_train_fp32_dk python tools/ncu_train_target.py 2 split fp32 > /dev/null 2>&1
$N --set full --import-source on --kernel-name-base demangled -k "regex:rgemm_kernel.*\(bool\)1, \(bool\)0>" -s 1 -c 1 -o $O/r5_train_fp32_coef python tools/ncu_train_target.py 2 split fp32 > /dev/null 2>&1
$N --set full --import-source on -k regex:stft_gemm_kernel -s 1 -c 1 -o $O/r5_mel_fp32 python tools/ncu_target.py mel 2 fp32 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_front -s 2 -c 1 -o $O/r5_cqt2010_front python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
$N --set full --import-source on -k regex:cqt2010_back -s 1 -c 1 -o $O/r5_cqt2010_back python tools/ncu_target.py cqt2010v2 2 f16 > /dev/null 2>&1
for w in "train fp32" "train tf32" "mel fp32" "stft fp32" "cqt2010v2 f16"; do set -- $w
  python bench.py --workload $1 --precision $2 > $O/r5_bench_$1_$2.json 2> $O/r5_bench_$1_$2.err
done
python tools/dbg_f16_chunk.py 1770 > $O/r5_f16_chunk.txt 2>&1
NNAB_RGEMM_F16_CHUNK=1024 python tools/dbg_f16_chunk.py 1770 >> $O/r5_f16_chunk.txt 2>&1
NNAB_RGEMM_F16_CHUNK=8192 python tools/dbg_f16_chunk.py 1770 >> $O/r5_f16_chunk.txt 2>&1
python tools/dbg_f16_dk.py 6 > $O/r5_f16_dk.txt 2>&1
ls -la $O | grep r5_
