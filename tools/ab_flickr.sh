for c in 16 10 5; do echo "== TOPK_CTAS_PER_SM=$c"; MAXK_TOPK_CTAS_PER_SM=$c bash tools/quick_times.sh flickr:32 reddit:32 products:32; done
for s in 1 4 16 32; do echo "== SCHED_CTRS=$s"; MAXK_SCHED_CTRS=$s bash tools/quick_times.sh flickr:32; done
