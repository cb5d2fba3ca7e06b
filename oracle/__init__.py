"""TEST INFRASTRUCTURE: the CPU oracle for the stage-1 path (see coral_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package, and only as the checker or the CPU baseline.
"""
