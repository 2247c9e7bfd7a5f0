timeout 600 python tools/ab_kernels.py C3 default rows_per_cta=148 rows_per_cta=37 items_per_thread=8 rows_per_cta=148,items_per_thread=8 rows_per_cta=296 2>&1 | grep '"db"'
timeout 600 python tools/ab_kernels.py C5 default items_per_thread=1 items_per_thread=2 items_per_thread=8 2>&1 | grep -E '"ctx_r"|"gelu"|"h1"|"probs_d"'
timeout 300 python tools/ab_kernels.py C4 default items_per_thread=1 items_per_thread=2 items_per_thread=8 2>&1 | grep '"y"'
