import sys, os
sys.path.insert(0, os.getcwd())
import paper_1205_4883_b200 as sv
lo, hi = (int(x) for x in os.environ.get("RANGE", "2,10000000001").split(","))
print(sv.stats(lo, hi))
