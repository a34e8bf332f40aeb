# per-wave times of library variants built under exp/*/ (and the shipped one):
#   bash tools/exp_waves.sh <config> <modes>     e.g. c5 baseline,live
shopt -s nullglob
cfg=${1:-c5}; modes=${2:-baseline}
for L in "" exp/*/libhrpp_b200.so; do
  echo "== ${L:-shipped} $cfg"
  HRPP_LIB=$L timeout 900 python tools/wave_times.py $cfg $modes 2>&1 | python -c "
import sys, json
tot = {}
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: print(line.rstrip()); continue
    tot.setdefault(d['mode'], []).append((d['wave'], d['ms'], d['bb']))
for m, w in tot.items():
    print(m, 'total %.3f ms' % sum(x[1] for x in w), ' '.join('%s=%.3f' % (a, b) for a, b, c in w), 'bb', sum(x[2] for x in w))
"
done
