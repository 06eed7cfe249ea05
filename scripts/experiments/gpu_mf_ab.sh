# matrix-free 3D 7-point K1 tile-shape A/B (abvar/m<TX>x<TY>)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in m32x8 m64x8 m32x16 m64x4 m128x4; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  echo "$v $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --operator stencil --config 7pt256 2>&1 >/dev/null | tail -1 | cut -c1-100)"
done; done
cp abvar/m64x8/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "matrix_free" 2>&1 | tail -2
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
