import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "tools")
from dense_bench import run
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
print(run(3, 64, reps, reps=2))
