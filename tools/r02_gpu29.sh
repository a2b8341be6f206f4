# round 2, GPU call 29 (box CPU only): the scheduler -> executor hand-off cost for RSim rows at G = 4
g++ -O2 -std=c++17 -pthread -Ipaper_2503_10516_b200/csrc tools/sched_prof.cpp paper_2503_10516_b200/csrc/sched.cpp paper_2503_10516_b200/csrc/sched_memo.cpp -o /tmp/sched_prof || exit 1
for i in 1 2 3; do
  /tmp/sched_prof rsim 4 0
  CEL_PROF_COPY=1 /tmp/sched_prof rsim 4 0
  CEL_PROF_QUEUE=1 /tmp/sched_prof rsim 4 0
  CEL_PROF_QUEUE=2 /tmp/sched_prof rsim 4 0
done
