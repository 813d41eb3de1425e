import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
from debug_parity import breakdown
for s in [(4,32,32,156,1,12,48),(16,16,16,156,1,12,48),(4,32,32,24,3,12,48),(4,32,32,24,6,12,48),(4,32,32,120,3,12,48),(4,16,16,24,12,12,48)]:
    breakdown(s, "fp32")
