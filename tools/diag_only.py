import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "tools")
from dense_bench import run
print(run(3, 64, 1, reps=2))
