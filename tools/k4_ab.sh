# K4 decode-step A/B between library builds (interleaved runs of tools/bench_step.py)
#   bash tools/k4_ab.sh rounds a.so b.so ...
R=$1; shift
for r in $(seq $R); do for L in "$@"; do
  echo -n "$(basename $L) "; RELAY_LIB=$L python tools/bench_step.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cold %.2f us hot %.2f us' % (d['cold']['us_per_step'], d['hot']['us_per_step']))"
done; done
