# device index sets: tests + timing vs host at cfg5; VMM probe
OUT=gpurun_out/${1:-r2d}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_index_device.py -q -x -rxXs > $OUT/pytest_index.log 2>&1; echo "pytest exit $?"; tail -5 $OUT/pytest_index.log
for a in "20 2 0" "20 2 1" "20 32 0" "20 32 1" "20 256 0"; do timeout 300 ./tools/vmm_probe $a; done > $OUT/vmm.log 2>&1; cat $OUT/vmm.log
timeout 600 python - > $OUT/index_time.log 2>&1 <<'PY'
import time, numpy as np, torch
torch.zeros(1, device="cuda")
import paper_2001_07289_b200 as P
mesh = P.build_mesh(3, (256, 256, 256), "p1")
theta = P.partition_uniform(mesh, (32, 32, 32))
for dev in (0, 0, None):
    pair = P.refine_uniform(mesh, theta, 2, validate=False)
    t0 = time.perf_counter(); o = P.classify_objects(pair, device=dev); t1 = time.perf_counter()
    w = P.compute_weights(pair, "cardinality", P.make_constant(mesh, 1.0), o); t2 = time.perf_counter()
    print("device" if dev is not None else "host", "classify %.3f s weights %.3f s objects %d" % (t1 - t0, t2 - t1, len(o)), flush=True)
    if dev is None: ref = o
    else: od = o
for f in ("signature", "owners", "kind", "dof_ptr", "dof_list", "dof_obj"):
    assert np.array_equal(getattr(od, f), getattr(ref, f)), f
print("cfg5 device == host")
PY
echo "index time exit $?"; cat $OUT/index_time.log
