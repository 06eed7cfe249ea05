for w in 1 2 3 4 8; do for c in 7pt256 27pt256; do
RVK_MF_WAVES=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --operator stencil --config $c > /dev/null 2> /tmp/e.err; echo "waves=$w $c $(tail -1 /tmp/e.err)"
done; done
