import ctypes as C, sys
sys.path.insert(0, ".")
lib = C.CDLL("paper_2112_06630_b200/lib/libknng_diag.so")
t = C.c_double(); ms = C.c_double(); t2 = C.c_double()
print("ffma", lib.knng_diag_ffma_peak(0, C.byref(t), C.byref(ms)), t.value, "ffma2", lib.knng_diag_ffma2_peak(0, C.byref(t2)), t2.value)
