"""Host-side logic of libsincos_pairs.so (validation, sharder, workspace sizing,
status strings) driven without a GPU, for a build with -fsanitize=address,undefined; run by
tests/test_sanitize_host.py with libasan/libubsan preloaded.  argv[1] = the library."""
import ctypes
import sys

L = ctypes.CDLL(sys.argv[1])
P, S, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
L.sincos_pairs.argtypes = [P, P, P, P, S, I, P]
buf = ctypes.create_string_buffer(4096)
a = ctypes.addressof(buf)
bad = 0
# validation paths (return before any CUDA call)
bad += L.sincos_pairs(a, None, None, None, 10, 0, None) != 1          # no output form
bad += L.sincos_pairs(a, a + 64, a + 128, a + 256, 10, 0, None) != 1   # both forms
bad += L.sincos_pairs(a, a + 64, a + 128, None, 10, 7, None) != 1     # bad variant
bad += L.sincos_pairs(a + 1, a + 64, a + 128, None, 10, 0, None) != 1 # misaligned
bad += L.sincos_pairs(a, a + 4, a + 128, None, 10, 0, None) != 2      # overlap
bad += L.sincos_pairs(a, a + 64, a + 68, None, 10, 0, None) != 2      # sin/cos overlap
bad += L.sincos_pairs(None, None, None, None, 0, 0, None) != 0        # n = 0
bad += L.sincos_pairs(a, a + 64, a + 128, None, (1 << 62), 0, None) != 1   # n too large
lo, hi = S(), S()
L.sincos_shard_range.argtypes = [S, I, I, ctypes.POINTER(S), ctypes.POINTER(S)]
for n in (0, 1, 7, 8, 1001, 1 << 40, (1 << 64) - 1):
    for G in (1, 2, 3, 8, 64):
        for g in range(G):
            bad += L.sincos_shard_range(n, G, g, ctypes.byref(lo), ctypes.byref(hi)) != 0
            bad += not (lo.value <= hi.value <= n)
bad += L.sincos_shard_range(10, 0, 0, ctypes.byref(lo), ctypes.byref(hi)) != -1
L.sincos_nudft_workspace_bytes.argtypes = [S, S]; L.sincos_nudft_workspace_bytes.restype = S
for nf, nt in ((0, 0), (0, 9), (9, 0), (1, 1), (1 << 20, 1 << 30), ((1 << 40), 3)):
    L.sincos_nudft_workspace_bytes(nf, nt)
L.sincos_status_string.restype = ctypes.c_char_p
for k in range(-1, 7):
    L.sincos_status_string(k)
print("san_abi", "ok" if bad == 0 else f"FAIL {bad}")
sys.exit(1 if bad else 0)
