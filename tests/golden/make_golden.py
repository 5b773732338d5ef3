"""Generate tests/golden/golden.npz — an INDEPENDENT torch-CPU restatement of
the SubNetAct operators and supernets, used to pin the C oracle.

The reference (servesim) has no tensor operators, so there are no
reference golden vectors for this path.  These fixtures come from a third,
independent implementation: numpy for the ssn_rng.h synthetic-data spec, and
torch.nn.functional (conv2d on OIHW weight slices, avg/max pools, batch-norm
with batch statistics for SubnetNorm calibration) for the networks of
DESIGN.md §3.  Regenerate with:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

torch.set_num_threads(8)
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# ---------------------------------------------------------------- ssn_rng.h
def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def u01(seed, kind, ordinal, idx):
    stream = np.array([(kind << 32) | ordinal], dtype=np.uint64)
    key = mix64(np.array([seed], dtype=np.uint64) ^ mix64(stream))
    with np.errstate(over="ignore"):
        h = mix64(key + np.asarray(idx, dtype=np.uint64) * np.uint64(0xD1B54A32D192ED03))
    return ((h >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)).astype(np.float32)


def bf16_round(a):
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32)


def weight(seed, ordinal, shape, bf16):
    n = int(np.prod(shape))
    fan_in = int(np.prod(shape[1:]))
    v = np.sqrt(np.float32(6.0) / np.float32(fan_in)) * (2 * u01(seed, 1, ordinal, np.arange(n)) - 1)
    v = v.astype(np.float32).reshape(shape)
    return bf16_round(v) if bf16 else v


def images(seed, ordinal, n, hw):
    return (2 * u01(seed, 5, ordinal, np.arange(n * 3 * hw * hw)) - 1).reshape(n, 3, hw, hw)


def md8(v):
    nv = max(8, int(v + 4) // 8 * 8)
    return nv + 8 if nv < 0.9 * v else nv


# ---------------------------------------------------------------- networks
class Net:
    """Holds weights in canonical ordinal order; runs a subnet forward."""

    def __init__(self, seed, bf16):
        self.seed, self.bf16 = seed, bf16
        self.w, self.g, self.b, self.bias = [], [], [], []
        self.bias_of = {}  # tensor ordinal -> bias

    def tensor(self, shape, linear=False):
        o = len(self.w)
        self.w.append(torch.from_numpy(weight(self.seed, o, shape, self.bf16)))
        if linear:
            self.bias.append(torch.from_numpy(0.1 * (2 * u01(self.seed, 4, o, np.arange(shape[0])) - 1)))
            self.bias_of[o] = self.bias[-1]
        return o

    def norm(self, c, res=False):
        o = len(self.g)
        u = u01(self.seed, 2, o, np.arange(c))
        self.g.append(torch.from_numpy(0.2 * u if res else 0.5 + u))
        self.b.append(torch.from_numpy(0.1 * (2 * u01(self.seed, 3, o, np.arange(c)) - 1)))
        return o


class Run:
    def __init__(self, net, calibrate, stats=None):
        self.net, self.calibrate = net, calibrate
        self.means, self.vars = [], []
        self.stats = stats
        self.cursor = 0

    def conv_bn(self, x, t, n, k, stride, cout, groups=1, res=None, relu=True, res_post=False):
        w = self.net.w[t]
        cin = x.shape[1]
        kmax = w.shape[2]
        off = (kmax - k) // 2
        if groups == 1:
            ws = w[:cout, :cin, off:off + k, off:off + k]
        else:
            ws = w[:cout, :, off:off + k, off:off + k]
        y = F.conv2d(x, ws, stride=stride, padding=k // 2, groups=groups)
        g, b = self.net.g[n][:cout], self.net.b[n][:cout]
        if self.calibrate:
            mu = y.mean(dim=(0, 2, 3))
            var = ((y - mu[None, :, None, None]) ** 2).mean(dim=(0, 2, 3))
            self.means.append(mu)
            self.vars.append(var)
        else:
            mu = self.stats[0][self.cursor:self.cursor + cout]
            var = self.stats[1][self.cursor:self.cursor + cout]
            self.cursor += cout
        y = (y - mu[None, :, None, None]) / torch.sqrt(var[None, :, None, None] + 1e-5)
        y = y * g[None, :, None, None] + b[None, :, None, None]
        if res is not None and not res_post:
            y = y + res
        if relu:
            y = torch.relu(y)
        if res is not None and res_post:
            y = y + res
        return y


def tinycnn(seed):
    net = Net(seed, bf16=False)
    base = [32, 32, 64, 128]
    blocks = [(0, 1, -1, 0), (0, 1, 0, 1), (0, 1, 1, 1), (1, 2, -1, 0), (1, 1, 2, 1), (1, 1, 3, 1),
              (2, 2, -1, 0), (2, 1, 4, 1)]
    spec = {"stem": (net.tensor((32, 3, 3, 3)), net.norm(32))}
    cin = 32
    spec["blocks"] = []
    for st, stride, flag, res in blocks:
        cout = base[1 + st]
        hid = md8(round(cin * 6.0))
        t1, n1 = net.tensor((hid, cin, 1, 1)), net.norm(hid)
        t2, n2 = net.tensor((hid, 1, 3, 3)), net.norm(hid)
        t3, n3 = net.tensor((cout, hid, 1, 1)), net.norm(cout, res=bool(res))
        spec["blocks"].append((st, stride, flag, res, t1, n1, t2, n2, t3, n3))
        cin = cout
    spec["fc"] = net.tensor((10, 128, 1, 1), linear=True)

    def forward(run, cfg, x):
        D, E, W = cfg
        C = [md8(base[i] * W[i]) for i in range(4)]
        y = run.conv_bn(x, *spec["stem"], 3, 1, C[0])
        for st, stride, flag, res, t1, n1, t2, n2, t3, n3 in spec["blocks"]:
            if flag >= 0 and not D[flag]:
                continue
            hid = md8(round(y.shape[1] * E[st]))
            h = run.conv_bn(y, t1, n1, 1, 1, hid)
            h = run.conv_bn(h, t2, n2, 3, stride, hid, groups=hid)
            y = run.conv_bn(h, t3, n3, 1, 1, C[1 + st], res=y if res else None, relu=False)
        g = y.mean(dim=(2, 3))
        w = net.w[spec["fc"]][:, :g.shape[1], 0, 0]
        return g @ w.T + net.bias[0]
    return forward, net


def resnet50(seed):
    net = Net(seed, bf16=True)
    SW, BD, NB = [256, 512, 1024, 2048], [2, 2, 4, 2], [4, 4, 6, 4]
    spec = {"stem": [(net.tensor((32, 3, 3, 3)), net.norm(32)),
                     (net.tensor((32, 32, 3, 3)), net.norm(32, True)),
                     (net.tensor((64, 32, 3, 3)), net.norm(64))]}
    cin, blocks = 64, []
    for s in range(4):
        mid = md8(round(SW[s] * 0.35))
        for bi in range(NB[s]):
            ds = (net.tensor((SW[s], cin, 1, 1)), net.norm(SW[s])) if bi == 0 else None
            a = (net.tensor((mid, cin, 1, 1)), net.norm(mid))
            b = (net.tensor((mid, mid, 3, 3)), net.norm(mid))
            c = (net.tensor((SW[s], mid, 1, 1)), net.norm(SW[s], True))
            blocks.append((s, bi, ds, a, b, c))
            cin = SW[s]
    fc = net.tensor((1000, 2048, 1, 1), linear=True)

    def forward(run, cfg, x):
        D, E, W = cfg
        mid_a = md8(md8(64 * W[0]) // 2)
        out_a = md8(64 * W[1])
        y = run.conv_bn(x, *spec["stem"][0], 3, 2, mid_a)
        if D[0]:
            y = run.conv_bn(y, *spec["stem"][1], 3, 1, mid_a, res=y, res_post=True)
        y = run.conv_bn(y, *spec["stem"][2], 3, 1, out_a)
        y = F.max_pool2d(y, 3, 2, 1)
        for idx, (s, bi, ds, a, b, c) in enumerate(blocks):
            if bi >= BD[s] and not D[1 + 2 * s + bi - BD[s]]:
                continue
            o = md8(SW[s] * W[2 + s])
            m = md8(round(o * E[idx]))
            stride = 2 if (s > 0 and bi == 0) else 1
            if ds is not None:
                p = F.avg_pool2d(y, stride, stride, ceil_mode=True) if stride > 1 else y
                r = run.conv_bn(p, ds[0], ds[1], 1, 1, o, relu=False)
            else:
                r = y
            h = run.conv_bn(y, a[0], a[1], 1, 1, m)
            h = run.conv_bn(h, b[0], b[1], 3, stride, m)
            y = run.conv_bn(h, c[0], c[1], 1, 1, o, res=r)
        g = y.mean(dim=(2, 3))
        w = net.w[fc][:, :g.shape[1], 0, 0]
        return g @ w.T + net.bias[0]
    return forward, net


def hswish(x):
    return x * torch.clamp(x + 3, 0, 6) / 6


def mbv3(seed):
    """OFA-MobileNetV3 w1.2 (DynamicMBConvLayer, DynamicSE), bf16-valued weights."""
    net = Net(seed, bf16=True)
    W, S, A, SE = [32, 48, 96, 136, 192], [2, 2, 2, 1, 2], [1, 1, 2, 2, 2], [0, 1, 0, 1, 1]
    first = (net.tensor((24, 3, 3, 3)), net.norm(24))
    fb = (net.tensor((24, 1, 3, 3)), net.norm(24), net.tensor((24, 24, 1, 1)), net.norm(24, True))
    cin, blocks = 24, []
    for st in range(5):
        for b in range(4):
            cout, stride = W[st], (S[st] if b == 0 else 1)
            res = stride == 1 and cin == cout
            mid = md8(round(cin * 6.0))
            ib = (net.tensor((mid, cin, 1, 1)), net.norm(mid))
            dw = (net.tensor((mid, 1, 7, 7)), net.norm(mid))
            se = None
            if SE[st]:
                sm = md8(mid // 4)
                se = (net.tensor((sm, mid, 1, 1), linear=True), net.tensor((mid, sm, 1, 1), linear=True))
            pl = (net.tensor((cout, mid, 1, 1)), net.norm(cout, res))
            blocks.append((st, b, stride, res, ib, dw, se, pl))
            cin = cout
    fe = (net.tensor((1152, 192, 1, 1)), net.norm(1152))
    fm = net.tensor((1536, 1152, 1, 1))
    net.tensor((1000, 1536, 1, 1), linear=True)  # classifier (weights last in net.w)
    fc = len(net.w) - 1

    def act(y, a):
        return torch.relu(y) if a == 1 else hswish(y)

    def forward(run, cfg, x):
        D, E, Wl, K = cfg
        biases = list(net.bias)  # linear tensors in ordinal order: SE pairs, then classifier
        y = act(run.conv_bn(x, *first, 3, 2, 24, relu=False), 2)
        h = run.conv_bn(y, fb[0], fb[1], 3, 1, 24, groups=24)
        y = run.conv_bn(h, fb[2], fb[3], 1, 1, 24, res=y, relu=False)
        se_i = 0
        for idx, (st, b, stride, res, ib, dw, se, pl) in enumerate(blocks):
            if se is not None:
                se_biases = (biases[se_i], biases[se_i + 1])
                se_i += 2
            if b >= 2 and not D[2 * st + b - 2]:
                continue
            mid = md8(round(y.shape[1] * E[idx]))
            h = act(run.conv_bn(y, ib[0], ib[1], 1, 1, mid, relu=False), A[st])
            h = act(run.conv_bn(h, dw[0], dw[1], K[idx], stride, mid, groups=mid, relu=False), A[st])
            if se is not None:
                C = h.shape[1]
                m = md8(C // 4)
                wr = net.w[se[0]][:m, :C, 0, 0]
                we = net.w[se[1]][:C, :m, 0, 0]
                p = h.mean(dim=(2, 3))
                s1 = torch.relu(p @ wr.T + se_biases[0][:m])
                s2 = torch.clamp(s1 @ we.T + se_biases[1][:C] + 3, 0, 6) / 6
                h = h * s2[:, :, None, None]
            y = run.conv_bn(h, pl[0], pl[1], 1, 1, W[st], res=y if res else None, relu=False)
        y = hswish(run.conv_bn(y, *fe, 1, 1, 1152, relu=False))
        g = y.mean(dim=(2, 3))
        f = hswish(g @ net.w[fm][:, :, 0, 0].T)
        return f @ net.w[fc][:, :, 0, 0].T + biases[-1]
    return forward, net


def bert(seed, classes):
    """Config 5: DynaBERT-style width/depth-sliced BERT-base."""
    net = Net(seed, True)
    t_tok, t_pos, t_typ = net.tensor((30522, 768)), net.tensor((512, 768)), net.tensor((2, 768))
    n_emb = net.norm(768)
    layers = []
    for _ in range(12):
        q, k, v, o = (net.tensor((768, 768), True) for _ in range(4))
        n1 = net.norm(768)
        f1, f2 = net.tensor((3072, 768), True), net.tensor((768, 3072), True)
        layers.append((q, k, v, o, n1, f1, f2, net.norm(768)))
    t_pool, t_cls = net.tensor((768, 768), True), net.tensor((classes, 768), True)

    def lin(x, t, cout, cin=None):
        w = net.w[t][:cout, :x.shape[-1] if cin is None else cin]
        return F.linear(x, w, net.bias_of[t][:cout])

    def ln(x, n):
        return F.layer_norm(x, (768,), net.g[n], net.b[n], eps=1e-12)

    def forward(cfg, ids):
        flags, (fe,), (hw,) = cfg
        heads = max(1, int(np.round(12 * hw)))
        ffn = min(3072, md8(3072 * fe))
        ca = heads * 64
        ids = torch.from_numpy(ids.astype(np.int64))
        nb, s = ids.shape
        x = net.w[t_tok][ids] + net.w[t_pos][:s][None] + net.w[t_typ][0][None, None]
        x = ln(x, n_emb)
        for on, (q, k, v, o, n1, f1, f2, n2) in zip(flags, layers):
            if not on:
                continue
            sp = lambda t: lin(x, t, ca).view(nb, s, heads, 64).transpose(1, 2)
            att = torch.softmax(sp(q) @ sp(k).transpose(-1, -2) / 8.0, dim=-1) @ sp(v)
            h = ln(lin(att.transpose(1, 2).reshape(nb, s, ca), o, 768) + x, n1)
            x = ln(lin(F.gelu(lin(h, f1, ffn)), f2, 768) + h, n2)
        pooled = torch.tanh(lin(x[:, 0], t_pool, 768))
        return lin(pooled, t_cls, classes)

    return forward


def tokens(seed, ordinal, n, s):
    return (u01(seed, 8, ordinal, np.arange(n * s)).astype(np.float64) * 30522).astype(
        np.int32).reshape(n, s)


def calibrate_and_forward(fwd, netobj, cfg, cal_x, x):
    r = Run(netobj, True)
    fwd(r, cfg, torch.from_numpy(cal_x))
    mean = torch.cat(r.means)
    var = torch.cat(r.vars)
    r2 = Run(netobj, False, (mean, var))
    logits = fwd(r2, cfg, torch.from_numpy(x))
    return mean.numpy(), var.numpy(), logits.numpy()


def main():
    out = {}
    seed = 0
    # ---- TinyCNN (config 1), reference default-catalog subnets + depth variants
    tiny_cfgs = [([True] * 5, [3.0, 4.0, 6.0], [w] * 4) for w in (0.4, 0.5, 0.6, 0.7, 0.85, 1.0)]
    tiny_cfgs += [([False, True, False, True, False], [3.0, 4.0, 6.0], [0.6] * 4),
                  ([False] * 5, [2.0, 3.0, 4.0], [0.4, 0.7, 0.5, 1.0])]
    fwd, netobj = tinycnn(seed)
    cal_x, x = images(seed, 100, 8, 32), images(seed, 1, 8, 32)
    for i, cfg in enumerate(tiny_cfgs):
        m, v, lg = calibrate_and_forward(fwd, netobj, cfg, cal_x, x)
        out[f"tiny{i}_mean"], out[f"tiny{i}_var"], out[f"tiny{i}_logits"] = m, v, lg
    out["tiny_cfgs"] = np.array(repr(tiny_cfgs))
    # ---- OFA-ResNet50 (config 2) at 32x32, bf16-valued weights, fp32 compute
    r50_cfgs = {
        "min": ([False] * 9, [0.2] * 18, [0.65] * 6),
        "max": ([True] * 9, [0.35] * 18, [1.0] * 6),
        "mixed": ([True, False, False, True, False, True, True, False, False],
                  [0.2, 0.35, 0.25] * 6, [1.0, 0.65, 0.8, 1.0, 0.65, 0.8]),
    }
    fwd, netobj = resnet50(seed)
    cal_x, x = images(seed, 100, 8, 32), images(seed, 1, 4, 32)
    for name, cfg in r50_cfgs.items():
        m, v, lg = calibrate_and_forward(fwd, netobj, cfg, cal_x, x)
        out[f"r50_{name}_mean"], out[f"r50_{name}_var"], out[f"r50_{name}_logits"] = m, v, lg
    out["r50_cfgs"] = np.array(repr(r50_cfgs))
    # ---- OFA-MobileNetV3 w1.2 (config 3) at 64x64
    mb_cfgs = {
        "min": ([False] * 10, [3.0] * 20, [1.0], [3] * 20),
        "max": ([True] * 10, [6.0] * 20, [1.0], [7] * 20),
        "mixed": ([True, False] * 5, [3.0, 4.0, 6.0, 4.0] * 5, [1.0], [3, 5, 7, 5] * 5),
    }
    fwd, netobj = mbv3(seed)
    cal_x, x = images(seed, 100, 8, 64), images(seed, 1, 4, 64)
    for name, cfg in mb_cfgs.items():
        m, v, lg = calibrate_and_forward(fwd, netobj, cfg, cal_x, x)
        out[f"mb_{name}_mean"], out[f"mb_{name}_var"], out[f"mb_{name}_logits"] = m, v, lg
    out["mb_cfgs"] = np.array(repr(mb_cfgs))
    # ---- width/depth-sliced BERT (config 5), seq 32, 4 classes, bf16-valued weights
    bert_cfgs = {
        "min": ([i not in (1, 3, 5, 7, 9, 11) for i in range(12)], [0.25], [0.25]),
        "mid": ([i not in (3, 7, 11) for i in range(12)], [0.5], [0.5]),
        "max": ([True] * 12, [1.0], [1.0]),
    }
    fwd = bert(seed, 4)
    ids = tokens(seed, 1, 2, 32)
    out["bert_ids"] = ids
    with torch.no_grad():
        for name, cfg in bert_cfgs.items():
            out[f"bert_{name}_logits"] = fwd(cfg, ids).numpy()
    out["bert_cfgs"] = np.array(repr(bert_cfgs))
    # ---- operator fixtures: WeightSlice conv with slices, crop, depthwise
    rng = np.random.default_rng(0)
    ops = []
    for (n, h, cin, cin_max, cout, cout_max, kmax, k, stride, dw) in [
            (2, 9, 12, 16, 20, 24, 3, 3, 1, False), (2, 10, 16, 16, 8, 32, 5, 3, 2, False),
            (1, 7, 24, 32, 24, 32, 7, 5, 1, True), (3, 6, 8, 8, 40, 48, 1, 1, 1, False)]:
        xo = rng.standard_normal((n, cin, h, h)).astype(np.float32)
        wshape = (cout_max, 1, kmax, kmax) if dw else (cout_max, cin_max, kmax, kmax)
        wo = rng.standard_normal(wshape).astype(np.float32)
        off = (kmax - k) // 2
        ws = torch.from_numpy(wo)[:cout, :(1 if dw else cin), off:off + k, off:off + k]
        y = F.conv2d(torch.from_numpy(xo), ws, stride=stride, padding=k // 2,
                     groups=cin if dw else 1)
        i = len(ops)
        out[f"op{i}_x"], out[f"op{i}_w"], out[f"op{i}_y"] = xo, wo, y.numpy()
        ops.append((n, h, cin, cin_max, cout, cout_max, kmax, k, stride, int(dw)))
    out["op_meta"] = np.array(ops, dtype=np.int64)
    out["rng_u01_first"] = u01(seed, 5, 0, np.arange(16))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
