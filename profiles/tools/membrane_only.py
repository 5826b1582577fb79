"""Run only the bench membrane leg (outer diffusion + porous inner steps);
prints its JSON object.  Used for profiling: python profiles/tools/membrane_only.py [steps]"""
import json, sys, types
sys.path.insert(0, '.')
import bench
args = types.SimpleNamespace(steps=int(sys.argv[1]) if len(sys.argv) > 1 else 20, warmup=3,
                             membrane_side=0.14)
print(json.dumps(bench.membrane_leg(args)))
