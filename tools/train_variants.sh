cp paper_2212_10550_b200/lib/libarfx.so /tmp/libarfx.keep
for v in paper_2212_10550_b200/lib/variants/*.so; do
  cp "$v" paper_2212_10550_b200/lib/libarfx.so
  n=$(basename "$v" .so)
  python -c "
import sys; sys.path.insert(0,'.')
import bench, json
from paper_2212_10550_b200._lib import lib, check
import ctypes as C
L=lib(); p64,p32=C.c_double(),C.c_double(); check(L.arfx_pipe_peaks(C.byref(p64),C.byref(p32)))
rk, ms, cnt = bench.bench_train_roofline(48, {'hbm_gbs':6553}, 'x', (p64.value,p32.value))
full = bench.bench_train_full(200)
print('$n', round(ms*1000,1), 'us/step seq;', {k: round(v['ms_per_launch']*1000,1) for k,v in rk.items() if k.startswith('bwd')}, 'pipelined it/s', round(full['iters_per_s']))
"
done
cp /tmp/libarfx.keep paper_2212_10550_b200/lib/libarfx.so
