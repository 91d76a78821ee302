# ncu --set full of each config's step kernel (one launch, after warm-up), CUDA
# events timing of the same command first.  Usage: bash tools/ncu_configs.sh <tag> [cases]
T=${1:-r2}
O=gpurun_out/$T
mkdir -p $O
for c in ${2:-c1 c2 c3 c4}; do
  F="--fma"; [ $c = c1 ] && F=""
  R=40; [ $c = c1 ] && R=1000; [ $c = c2 ] && R=200
  timeout 300 python tools/prof_cases.py $c --reps $R $F > $O/$c.json 2>&1 || continue
  case $c in
    c1) K="regex:ring_lin"; S=1 ;;
    c2) K="regex:etd2_persist"; S=1 ;;
    *) K="regex:step_kernel"; S=3 ;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k $K -s $S -c 1 -o $O/$c \
    python tools/prof_cases.py $c --reps $R $F > $O/ncu_$c.log 2>&1
  echo "$c ncu rc=$?"
done
ls $O
