import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1511_03645_b200 import _lib
print(json.dumps(bench.bench_c5_full(int(sys.argv[1]) if len(sys.argv) > 1 else 9, _lib.VARIANT_FAST)))
