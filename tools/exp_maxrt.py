"""Experiment (GPU box): repeat the bench's max-real-time search at the c3
shape a few times to see its run-to-run spread at the threshold."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for r in range(reps):
    m = bench.max_realtime(A, dict(bench.CONFIGS["c3"]), 0, budget_s=110.0)
    print(json.dumps({"rep": r, "channels": m["channels"],
                      "trials": [(t["L"], t.get("device_p99_us") and round(t["device_p99_us"], 1),
                                  t.get("paced_e2e_p99_us") and round(t["paced_e2e_p99_us"], 1))
                                 for t in m["trials"]][-4:]}), flush=True)
