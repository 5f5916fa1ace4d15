import sys, json, time
sys.path.insert(0,'.')
import bench, paper_1912_06127_b200 as pkg
t0=time.time(); r=bench.secondary_u1(pkg, 2, 1); print(json.dumps(r)[:1500]); print('wall', time.time()-t0)
