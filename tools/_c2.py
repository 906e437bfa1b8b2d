import json, sys
sys.path.insert(0, ".")
import bench
from tools import dlrm_secondary as DS
from paper_2104_09455_b200 import netprofile as NP
r = DS.run(NP.device_profile(bench.load_peaks()[0]), steps=20, warmup=3)
print(json.dumps(r))
