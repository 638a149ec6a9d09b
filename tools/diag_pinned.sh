free -g; ulimit -l; for n in /sys/devices/system/node/node*/meminfo; do grep -E "MemTotal|MemFree" $n; done; nproc
python - <<'PY'
import sys, ctypes as C, time
sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C
lib = _C.lib()
for gb in (8, 16, 32, 48):
    for node in (-1, 0, 1):
        p = C.c_void_p()
        t = time.time()
        rc = lib.pm_host_alloc_numa(C.c_ulonglong(gb << 30), node, C.byref(p))
        dt = time.time() - t
        print(f"{gb} GB node {node}: rc={rc} {dt:.1f}s", flush=True)
        if rc == 0:
            lib.pm_host_free_numa(p, C.c_ulonglong(gb << 30), node)
PY
free -g
