# A/B of prebuilt library variants on one box: abvar/<name>/librvk.so swapped in
# turn; CFGS (default 7pt256) = bench configs, ROUNDS (default 2) repetitions,
# BENCH_ARGS = extra bench.py arguments (e.g. --mode persistent)
for r in $(seq ${ROUNDS:-2}); do for c in ${CFGS:-7pt256}; do for v in "$@"; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  echo "$c $v $(python bench.py --no-cpu-baseline --no-strong --steps 20 --config $c $BENCH_ARGS 2>&1 >/dev/null | tail -1 | cut -c1-90)"
done; done; done
