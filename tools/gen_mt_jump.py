"""Generates paper_1508_03110_b200/csrc/mt_jump_table.inc: jump-ahead polynomials of mt19937_64.

The device x0 generator (k_vec.cu) splits the draw stream into chunks of L = 312*256 draws and
needs the generator state at every chunk start.  With T the one-step transition of the 19937-bit
state, T^J s = g_J(T) s for g_J(x) = x^J mod phi(x), phi the characteristic polynomial of T
(Haramoto, Matsumoto, Nishimura, Panneton, L'Ecuyer: "Efficient jump ahead for F2-linear random
number generators", 2008).  g_J(T) s = XOR over the set coefficients i of the state window at i.

This script
  1. finds phi by Berlekamp-Massey on one state bit of the word sequence (degree must be 19937),
  2. computes g_J for J = L, 8L, 64L, 512L by square-and-multiply modulo phi,
  3. checks every g_J against stepping the generator J draws from a test seed,
  4. writes the four polynomials as 312 little-endian 64-bit words each.

  python tools/gen_mt_jump.py            # ~1-2 minutes
"""
import os
import sys

N, M = 312, 156
A = 0xB5026F5AA96619E9
UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
MASK = (1 << 64) - 1
DEG = 19937
L = 312 * 256
JUMPS = [L, 8 * L, 64 * L, 512 * L]


def seed_state(seed):
    st = [seed & MASK]
    for i in range(1, N):
        st.append((6364136223846793005 * (st[-1] ^ (st[-1] >> 62)) + i) & MASK)
    return st


def words(state, count):
    """w_0 .. w_{count-1}: the untempered word sequence continuing `state` (w_0..w_311)."""
    w = list(state)
    while len(w) < count:
        k = len(w) - N
        y = (w[k] & UM) | (w[k + 1] & LM)
        w.append(w[k + M] ^ (y >> 1) ^ (A if y & 1 else 0))
    return w[:count]


def bit_reverse(poly, width):
    """bit j of poly -> bit (width - j), j = 0..width."""
    return int(bin(poly & ((1 << (width + 1)) - 1))[2:].zfill(width + 1)[::-1], 2)


def berlekamp_massey(bits):
    """Connection polynomial C (int, bit j = c_j, c_0 = 1) and linear complexity Lc of a GF(2)
    sequence: s_i = sum_{j=1..Lc} c_j s_{i-j}."""
    s = 0  # bit i of s = bits[i]
    for i, b in enumerate(bits):
        if b:
            s |= 1 << i
    C, B, Lc, m = 1, 1, 0, 1
    for i in range(len(bits)):
        # discrepancy d = sum_{j=0..Lc} c_j s_{i-j}: c reversed over Lc+1 bits against s_{i-Lc..i}
        lo = max(i - Lc, 0)
        width = i - lo
        d = bin(((s >> lo) & ((1 << (width + 1)) - 1)) & bit_reverse(C, width)).count("1") & 1
        if d == 0:
            m += 1
        elif 2 * Lc <= i:
            C, B = C ^ (B << m), C
            Lc = i + 1 - Lc
            m = 1
        else:
            C ^= B << m
            m += 1
    return C, Lc


def mulmod(a, b, phi):
    r = 0
    top = 1 << DEG
    for i in range(b.bit_length() - 1, -1, -1):
        r <<= 1
        if r & top:
            r ^= phi
        if (b >> i) & 1:
            r ^= a
    return r


def xpow(J, phi):
    r, base = 1, 2  # 1 and x
    e = J
    while e:
        if e & 1:
            r = mulmod(r, base, phi)
        base = mulmod(base, base, phi)
        e >>= 1
    return r


def jump(state, g):
    """g(T) applied to `state`: XOR of the windows at the set coefficients."""
    w = words(state, DEG + N)
    out = [0] * N
    i = 0
    gg = g
    while gg:
        if gg & 1:
            for k in range(N):
                out[k] ^= w[i + k]
        gg >>= 1
        i += 1
    return out


def same_state(a, b):
    return (a[0] & UM) == (b[0] & UM) and a[1:] == b[1:]


def read_table(path):
    """The polynomials of mt_jump_table.inc as ints."""
    import re
    nums = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ull", open(path).read())]
    assert len(nums) == len(JUMPS) * N
    return [sum(nums[p * N + k] << (64 * k) for k in range(N)) for p in range(len(JUMPS))]


def main():
    st = seed_state(5489)
    nb = 2 * DEG + 64
    w = words(st, nb)
    bits = [(x >> 63) & 1 for x in w]
    C, Lc = berlekamp_massey(bits)
    assert Lc == DEG, Lc
    # phi(x) = x^L * C(1/x): coefficient of x^(L-j) is c_j
    phi = bit_reverse(C, DEG)
    assert phi >> DEG == 1
    polys = []
    for J in JUMPS:
        g = xpow(J, phi)
        polys.append(g)
        print(f"x^{J} mod phi: weight {bin(g).count('1')}", flush=True)
    # checks: against stepping the generator (two seeds for the first, one for the rest but the last)
    for seed in (0, 12345):
        s0 = seed_state(seed)
        ref = words(s0, JUMPS[1] + N)
        assert same_state(jump(s0, polys[0]), ref[JUMPS[0]:JUMPS[0] + N])
        assert same_state(jump(s0, polys[1]), ref[JUMPS[1]:JUMPS[1] + N])
    s0 = seed_state(7)
    ref = words(s0, JUMPS[2] + N)
    assert same_state(jump(s0, polys[2]), ref[JUMPS[2]:JUMPS[2] + N])
    # the last by composition: x^(512L) = (x^(64L))^8
    g = polys[2]
    for _ in range(3):
        g = mulmod(g, g, phi)
    assert g == polys[3]
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1508_03110_b200", "csrc",
                       "mt_jump_table.inc")
    with open(out, "w") as f:
        f.write("// Generated by tools/gen_mt_jump.py -- x^J mod phi(x) of mt19937_64 for J = L, 8L, 64L, 512L,\n"
                "// L = 312*256 draws; 312 little-endian 64-bit words per polynomial (bit i = coefficient of x^i).\n")
        for g in polys:
            f.write("{\n")
            for k in range(N):
                f.write(f"0x{(g >> (64 * k)) & MASK:016x}ull,")
                f.write("\n" if k % 4 == 3 else " ")
            f.write("},\n")
    print("wrote", os.path.normpath(out))


if __name__ == "__main__":
    main()
