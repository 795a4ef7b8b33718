"""bench.py's busyring measurement alone (HH + STDP workload, bench.cpp:134-194)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
print(json.dumps(bench.busyring_configs(), indent=1))
