timeout 900 python profiles/r02/chunk_model_ab.py 2>&1 | tail -12
