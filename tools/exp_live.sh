# per-wave live-mode times of library variants built under exp/*/ (and the shipped one):
#   bash tools/exp_live.sh <config> [mode]
shopt -s nullglob
for L in "" exp/*/libhrpp_b200.so; do
  echo -n "${L:-shipped} "
  HRPP_LIB=$L timeout 900 python tools/live_waves.py ${1:-c5} ${2:-live} 2>&1 | tail -1
done
