# round-1 profile set: one ncu --set full capture per workload's dominant kernel (+ baselines),
# then the launch list of the default bench command. Summarised by tools/make_profiles.py r01.
mkdir -p gpurun_out
cap() {  # name kernel-regex skip count env... -- prof_case args
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  timeout 900 env "$@" > /dev/null 2>&1
  :
}
run() {
  local name=$1 rx=$2 skip=$3 cnt=$4 envs=$5; shift 5
  env $envs timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c $cnt \
      -o gpurun_out/r01_$name python tools/prof_case.py "$@" > gpurun_out/r01_$name.log 2>&1
  tail -1 gpurun_out/r01_$name.log
}
run cfg2_spec k_spec 8 1 "CUPSO_SYNC_MODE=spec" cuda-sync cubic 20 1 600
run cfg2_sync k_sync_res 0 1 "CUPSO_SYNC_MODE=resident" cuda-sync cubic 20 1 200
run cfg2_reduction_step k_classic_step 5 1 "X=1" cuda-reduction cubic 20 1 10
run cfg2_reduction_fold k_classic_fold 5 1 "X=1" cuda-reduction cubic 20 1 10
run cfg3_async k_async_reg 0 1 "X=1" cuda-async cubic 24 1 100
run cfg4_spec k_spec 0 60 "CUPSO_SYNC_MODE=spec" cuda-sync rastrigin 20 32 60
run cfg4_f32 k_spec32_split 0 60 "X=1" cuda-sync-f32 rastrigin 20 32 60
run cfg4_wave k_wave 5 1 "CUPSO_SYNC_MODE=wave" cuda-sync rastrigin 20 32 10
run cfg5proxy_spec k_spec 0 40 "CUPSO_SYNC_MODE=spec" cuda-sync sphere 24 8 20
run cfg5proxy_wave k_wave 5 1 "CUPSO_SYNC_MODE=wave" cuda-sync sphere 24 8 10
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | wc -l
# summaries travel back; the large multi-launch reports do not (gpurun_out <= 64 MiB)
python tools/make_profiles.py r01 gpurun_out/profiles_r01
for f in gpurun_out/*.ncu-rep; do [ $(stat -c %s "$f") -gt 6000000 ] && rm -f "$f"; done
du -sh gpurun_out
