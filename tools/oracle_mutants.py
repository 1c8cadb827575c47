"""Mutation check of the oracle's pins (VERDICT r1 'What's weak' 1): apply each plausible slip to
a copy of oracle/dyllm_oracle.py, run the CPU suite, and report whether a pin catches it.
Restores the file afterwards.   python tools/oracle_mutants.py"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "oracle", "dyllm_oracle.py")
MUTANTS = {
    "dV sign flipped": ("dV = V[idx_in] - cache.V[idx_in]", "dV = cache.V[idx_in] - V[idx_in]"),
    "C = C_cache - dC": ("C = cache.C[input_rows] + dC", "C = cache.C[input_rows] - dC"),
    "C = C_cache + 0.5 dC": ("C = cache.C[input_rows] + dC", "C = cache.C[input_rows] + 0.5 * dC"),
    "ApproxAttn on pre-merge K": ("dC = approx_attention(q_in, K, dV", "dC = approx_attention(q_in, cache.K, dV"),
    "exact rows on pre-merge V": ("c_sal = attention(q_in[pos_in_input], K, V,", "c_sal = attention(q_in[pos_in_input], K, cache.V,"),
    "K not merged": ("        K[idx_in] = k_new\n", "        pass\n"),
    "lm_logits without final RMSNorm": ('return rms_norm(h, wg["g_final"], cfg.rms_eps) @ wg["lm_head"].T',
                                        'return h @ wg["lm_head"].T'),
    "residual_mode 1 without RMSNorm": ('h = rms_norm(o, w["g_ffn"], cfg.rms_eps)\n    return h, ffn(h, w)',
                                        'h = o\n    return h, ffn(h, w)'),
    "residual_mode 0 without FFN residual": ("return h, h + ffn(", "return h, ffn("),
    "softmax scale 1/hd": ("/ np.sqrt(head_dim)", "/ head_dim"),
    "RoPE sign": ("x2 * c + x1 * s", "x2 * c - x1 * s"),
    "select <= instead of <": ("(s <= tau) if cmp else (s < tau)", "(s <= tau) if cmp else (s <= tau)"),
    "C cache not committed": ("    cache.C[input_rows] = C\n", ""),
    "Q cache not refreshed": ("            q_in[where] = qr\n", ""),
    "cosine without sqrt": ("dot[i] / np.sqrt(na2[i] * nb2[i])", "dot[i] / (na2[i] * nb2[i])"),
    "unmask ties to highest position": ("key=lambda i: (-conf[i], cand_pos[i])", "key=lambda i: (-conf[i], -cand_pos[i])"),
    "layer-1 idx ignores decoded rows": ("base = np.union1d(base, st.decoded_prev)", "base = base"),
}


def main():
    src = open(PATH).read()
    backup = tempfile.mktemp()
    shutil.copy(PATH, backup)
    survived = []
    try:
        for name, (a, b) in MUTANTS.items():
            assert a in src, name
            open(PATH, "w").write(src.replace(a, b))
            r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests"), "-x", "-q", "-m",
                                "not gpu", "-p", "no:cacheprovider"], capture_output=True, text=True, cwd=ROOT)
            tail = r.stdout.strip().splitlines()[-1]
            print(f"{name:40s} {'caught' if r.returncode else 'SURVIVED'}  ({tail})", flush=True)
            if not r.returncode:
                survived.append(name)
    finally:
        shutil.copy(backup, PATH)
    print("survivors:", survived or "none")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
