for e in 16 0 16 0; do DG_EXP=$e python profiles/r02/cheb_time.py 2>&1 | grep DG_EXP; done
