#!/bin/bash
# compute-sanitizer over every kernel variant.  Logs -> gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool name env... -- mode
  local tool=$1 name=$2 mode=$3; shift 3
  echo "== $tool $name ($mode) env: $*" | tee -a $OUT/summary.txt
  env "$@" timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_workload.py $mode > $OUT/${tool}_${name}.log 2>&1
  echo "rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' $OUT/${tool}_${name}.log | tail -2 | tr '\n' ' ')" | tee -a $OUT/summary.txt
}
VARIANTS=("default:bn:X=0" "splitk:bn:SLIM_SPLITK_FORCE=1" "nohalo:bn:SLIM_NO_HALO=1"
  "halo_large_only:bn:SLIM_HALO_NO_S2=1 SLIM_HALO_NO_PROJ=1 SLIM_HALO_NO_SMALL=1"
  "x3_1:bn:SLIM_HALO_X3=1" "x3_2:bn:SLIM_HALO_X3=2" "stages1:bn:SLIM_HALO_STAGES=1 SLIM_HALO_EPI1=1"
  "narrow:bn:SLIM_HALO_NARROW=1" "nprod1:bn:SLIM_NPROD=1" "small:bn:SLIM_HALO_SMALL=1"
  "mc4:bn:SLIM_MC_MAX=4" "gn:gn:X=0" "fp32:fp32:X=0")
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  for v in "${VARIANTS[@]}"; do
    IFS=: read name mode envs <<< "$v"
    run $tool $name $mode $envs
  done
done
