// Circuit -> tensor network (Sec. II.B.1).
#include <cstdio>
#include <fstream>

#include "jt_internal.hpp"

using namespace jt;

namespace jt {

jt_network* network_create(int32_t n_wires, int32_t d) {
  if (n_wires < 1 || d < 2) fail(JT_EUSAGE, "jt_network_create: need n_wires >= 1 and d >= 2");
  auto* net = new jt_network();
  net->n_wires = n_wires;
  net->d = d;
  net->cur.resize(n_wires);
  for (int w = 0; w < n_wires; ++w) {  // |0>_w, rank 1 (l.81)
    HostTensor t;
    t.labels = {w};
    t.data.assign(d, cplx(0, 0));
    t.data[0] = 1.0;
    net->tensors.push_back(std::move(t));
    net->cur[w] = w;
  }
  net->n_labels = n_wires;
  return net;
}

void network_add_gate(jt_network* net, int32_t k, const int32_t* wires, const double* u) {
  if (!net || !wires || !u) fail(JT_EUSAGE, "jt_network_add_gate: null argument");
  if (net->closed) fail(JT_EVALIDATION, "jt_network_add_gate: network already closed");
  if (k != 1 && k != 2) fail(JT_EUSAGE, "jt_network_add_gate: k must be 1 or 2");
  for (int i = 0; i < k; ++i) {
    if (wires[i] < 0 || wires[i] >= net->n_wires) fail(JT_EUSAGE, "jt_network_add_gate: wire out of range");
    for (int j = 0; j < i; ++j)
      if (wires[j] == wires[i]) fail(JT_EUSAGE, "jt_network_add_gate: repeated wire");
  }
  const int64_t dim = (k == 1) ? net->d : int64_t(net->d) * net->d;
  HostTensor t;
  // labels (out_0..out_{k-1}, in_0..in_{k-1}), reading A7 (P:81 B_cfbe: outs c,f then ins b,e)
  std::vector<int64_t> outs(k), ins(k);
  for (int i = 0; i < k; ++i) {
    outs[i] = net->n_labels++;
    ins[i] = net->cur[wires[i]];
  }
  for (int i = 0; i < k; ++i) t.labels.push_back(outs[i]);
  for (int i = 0; i < k; ++i) t.labels.push_back(ins[i]);
  t.data.resize(dim * dim);
  for (int64_t i = 0; i < dim * dim; ++i) t.data[i] = cplx(u[2 * i], u[2 * i + 1]);
  for (int i = 0; i < k; ++i) net->cur[wires[i]] = outs[i];
  net->tensors.push_back(std::move(t));
  net->n_gates++;
}

void network_close(jt_network* net, const int32_t* x, const int32_t* open_wires, int32_t n_open) {
  if (!net || !x) fail(JT_EUSAGE, "jt_network_close: null argument");
  if (net->closed) fail(JT_EVALIDATION, "jt_network_close: already closed");
  if (n_open < 0 || n_open > net->n_wires || (n_open > 0 && !open_wires))
    fail(JT_EUSAGE, "jt_network_close_batch: bad open-wire list");
  std::vector<int> open_idx(net->n_wires, -1);
  for (int i = 0; i < n_open; ++i) {
    const int w = open_wires[i];
    if (w < 0 || w >= net->n_wires) fail(JT_EUSAGE, "jt_network_close_batch: open wire out of range");
    if (open_idx[w] >= 0) fail(JT_EUSAGE, "jt_network_close_batch: repeated open wire");
    open_idx[w] = i;
  }
  for (int w = 0; w < net->n_wires; ++w)
    if (open_idx[w] < 0 && (x[w] < 0 || x[w] >= net->d)) fail(JT_EUSAGE, "jt_network_close: digit out of range");
  net->batch_labels.assign(n_open, -1);
  for (int i = 0; i < n_open; ++i) net->batch_labels[i] = net->n_labels + i;
  for (int w = 0; w < net->n_wires; ++w) {
    HostTensor t;
    if (open_idx[w] < 0) {  // <x_w|, rank 1 (l.83)
      t.labels = {net->cur[w]};
      t.data.assign(net->d, cplx(0, 0));
      t.data[x[w]] = 1.0;
    } else {  // identity (wire label, batch label): the batch digit y selects <y|
      t.labels = {net->cur[w], net->batch_labels[open_idx[w]]};
      t.data.assign((size_t)net->d * net->d, cplx(0, 0));
      for (int y = 0; y < net->d; ++y) t.data[(size_t)y * net->d + y] = 1.0;
    }
    net->tensors.push_back(std::move(t));
  }
  net->n_labels += n_open;
  net->closed = true;
}

void network_export(const jt_network* net, const char* path) {
  std::ofstream f(path);
  if (!f) fail(JT_EUSAGE, std::string("cannot open ") + path);
  f << "{\"n_wires\": " << net->n_wires << ", \"d\": " << net->d << ", \"closed\": "
    << (net->closed ? "true" : "false") << ", \"n_labels\": " << net->n_labels << ", \"batch_labels\": [";
  for (size_t i = 0; i < net->batch_labels.size(); ++i) f << (i ? ", " : "") << net->batch_labels[i];
  f << "], \"tensors\": [";
  for (size_t t = 0; t < net->tensors.size(); ++t) {
    f << (t ? ", " : "") << "[";
    const auto& ls = net->tensors[t].labels;
    for (size_t i = 0; i < ls.size(); ++i) f << (i ? ", " : "") << ls[i];
    f << "]";
  }
  // tensor data, row-major over the labels in the order above, interleaved re, im (exact:
  // 17 significant digits round-trip a double)
  f << "], \"data\": [";
  f.precision(17);
  for (size_t t = 0; t < net->tensors.size(); ++t) {
    f << (t ? ", " : "") << "[";
    const auto& dv = net->tensors[t].data;
    for (size_t i = 0; i < dv.size(); ++i) f << (i ? ", " : "") << dv[i].real() << ", " << dv[i].imag();
    f << "]";
  }
  f << "]}\n";
}

}  // namespace jt
