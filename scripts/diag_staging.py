import sys, time
sys.path.insert(0, "/root/repo")
import paper_2604_01949_b200 as R
spec = "procedural:counts?n_obs=%s&n_var=36000&seed=1&chunk_rows=1024&chunks_per_shard=128" % sys.argv[1]
t = time.time()
try:
    ds = R.DeviceStore(R.StoreReader(spec), 0, sys.argv[2])
    print("ok", sys.argv, ds.image_bytes(), time.time() - t)
except Exception as e:
    print("FAIL", sys.argv, e, time.time() - t)
