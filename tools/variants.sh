# bench each prebuilt library variant in paper_2212_10550_b200/lib/variants/ (tuning runs)
cp paper_2212_10550_b200/lib/libarfx.so /tmp/libarfx.keep
for v in paper_2212_10550_b200/lib/variants/*.so; do
  cp "$v" paper_2212_10550_b200/lib/libarfx.so
  n=$(basename "$v" .so)
  timeout 240 python bench.py --no-cpu-baseline --no-extra --steps 60 > gpurun_out/var_$n.json 2> gpurun_out/var_$n.err
  echo "$n rc=$?"
done
cp /tmp/libarfx.keep paper_2212_10550_b200/lib/libarfx.so
