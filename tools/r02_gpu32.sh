# round 2, GPU call 32 (box CPU only): hand-off as a ring of reused slots vs a deque of copies
g++ -O2 -std=c++17 -pthread -Ipaper_2503_10516_b200/csrc tools/sched_prof.cpp paper_2503_10516_b200/csrc/sched.cpp paper_2503_10516_b200/csrc/sched_memo.cpp -o /tmp/sched_prof || exit 1
for i in 1 2 3; do
  /tmp/sched_prof rsim 4 0
  CEL_PROF_QUEUE=1 /tmp/sched_prof rsim 4 0
  CEL_PROF_QUEUE=3 /tmp/sched_prof rsim 4 0
done
