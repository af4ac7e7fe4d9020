// qsv_program: the compiled replacement of Circuit.update_state's per-gate
// loop (reference circuit.py:48-55).  Creation canonicalises every gate,
// copies all payloads to the device once and plans the steps; run replays the
// steps on the state's stream (optionally through a CUDA graph, which removes
// the per-launch CPU cost for small states).
#include <cstring>
#include <string>
#include <cmath>
#include <vector>
#include <algorithm>

#include "qsv_internal.cuh"
#include "qsv_program.cuh"
#include "qsv_tile.cuh"

using namespace qsv;

struct qsv_program {
  int n;
  std::vector<Step> steps;
  std::vector<TilePlan> tiles;
  void* dev_payload = nullptr;
  size_t payload_bytes = 0;
  int payload_device = -1;       // device holding dev_payload
  cudaEvent_t payload_ready = nullptr;  // the upload's completion (runs wait on it)
  std::vector<char> host_payload;  // re-uploaded when a state on another device runs it
  qsv_program_stats stats;
  qsv_plan_opts opts;
  // CUDA graph cache (valid for one amps pointer / stream / device)
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  double2* graph_amps = nullptr;
  unsigned long long* graph_ctr = nullptr;  // the captured tile passes' work counter
  cudaStream_t graph_stream = nullptr;
  int graph_sm_limit = 0;
  cudaStream_t last_stream = 0;  // the payload is released in this stream's order
  uint64_t runs = 0;
  int device = -1;
  bool jit_tried = false;  // generated pass kernels compiled / fetched
};

namespace {

int launch_steps(qsv_program* p, double2* amps, cudaStream_t s, int max_ctas,
                 unsigned long long* ctr, uint64_t fmask = 0, uint64_t fval = 0) {
  for (const Step& st : p->steps) {
    int rc;
    if (st.type == 0) {
      const Cplx* dev =
          st.has_payload ? reinterpret_cast<const Cplx*>((char*)p->dev_payload + st.payload_off)
                         : nullptr;
      rc = launch_gate(amps, p->n, st.gate, dev, s);
    } else {
      rc = launch_tile_pass(amps, p->n, p->tiles[st.tile], p->dev_payload, s, max_ctas, ctr,
                            fmask, fval);
    }
    if (rc) return rc;
  }
  return QSV_OK;
}

// A private non-blocking stream per device for payload uploads: the copy
// neither waits for nor blocks the work queued on the legacy / state streams
// (a synchronous cudaMemcpy would first drain the legacy stream, stalling the
// host behind every kernel queued so far -- e.g. the sharded engine compiling
// the next segment while the current exchange is still running).
cudaStream_t upload_stream(int dev) {
  static cudaStream_t streams[64] = {};
  if (dev < 0 || dev >= 64) return 0;
  if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  return streams[dev];
}

// payload on `dev` (programs are built on the current device; a state on
// another device triggers a re-upload there).  Asynchronous: runs wait on
// payload_ready; host_payload stays alive as the copy's source.
int upload_payload(qsv_program* p, int dev) {
  if (p->host_payload.empty() || p->payload_device == dev) return QSV_OK;
  if (p->dev_payload) {
    DeviceGuard old(p->payload_device);
    dev_free(p->dev_payload, p->payload_bytes, p->last_stream);
    p->dev_payload = nullptr;
  }
  if (p->payload_ready) {
    cudaEventDestroy(p->payload_ready);
    p->payload_ready = nullptr;
  }
  DeviceGuard dg(dev);
  cudaStream_t us = upload_stream(dev);
  cudaError_t e = dev_alloc(&p->dev_payload, p->payload_bytes, dev, us);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(program payload)");
  e = cudaMemcpyAsync(p->dev_payload, p->host_payload.data(), p->payload_bytes,
                      cudaMemcpyHostToDevice, us);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(program payload)");
  e = cudaEventCreateWithFlags(&p->payload_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(p->payload_ready, us);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(program payload)");
  p->payload_device = dev;
  p->last_stream = us;
  return QSV_OK;
}

// Compile (or fetch from the caches) the generated kernel of every tile pass
// that has one; passes whose compilation fails keep the interpreter.
int jit_prepare(qsv_program* p) {
  if (p->jit_tried) return QSV_OK;
  p->jit_tried = true;
  std::vector<const std::string*> srcs;
  std::vector<TilePlan*> tps;
  for (TilePlan& tp : p->tiles)
    if (!tp.jit_src.empty() && !tp.jit.kernel) {
      srcs.push_back(&tp.jit_src);
      tps.push_back(&tp);
    }
  if (srcs.empty()) return QSV_OK;
  std::vector<JitKernel> ks;
  std::string err;
  const int rc = jit_kernels(srcs, ks, &err);
  if (rc) return rc;
  int ok = 0;
  for (size_t i = 0; i < tps.size(); ++i) {
    tps[i]->jit = ks[i];
    if (ks[i].kernel) ++ok;
  }
  p->stats.num_jit_passes = ok;
  if (!err.empty() && getenv("QSV_JIT_VERBOSE")) fprintf(stderr, "qsv jit: %s\n", err.c_str());
  return QSV_OK;
}

bool jit_all_cached(const qsv_program* p) {
  bool any = false;
  for (const TilePlan& tp : p->tiles)
    if (!tp.jit_src.empty()) {
      any = true;
      if (!jit_cached(tp.jit_src)) return false;
    }
  return any;
}

// every pass's structure was planned before in this process (a parametric
// circuit recompiled with new angles, a shard segment seen before): worth
// compiling at creation even for a program that will run only once
bool jit_all_seen(const qsv_program* p) {
  bool any = false;
  for (const TilePlan& tp : p->tiles)
    if (!tp.jit_src.empty()) {
      any = true;
      if (!tp.jit_seen) return false;
    }
  return any;
}

void drop_graph(qsv_program* p) {
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->graph) cudaGraphDestroy(p->graph);
  p->gexec = nullptr;
  p->graph = nullptr;
  p->graph_amps = nullptr;
  p->graph_ctr = nullptr;
}

}  // namespace

static int convert_ops(int n, const qsv_op* ops, int nops, std::vector<GateDesc>& gates) {
  gates.reserve(nops);
  for (int i = 0; i < nops; ++i) {
    const qsv_op& op = ops[i];
    GateDesc g;
    memset(g.targets, 0, sizeof(g.targets));
    memset(g.ids, 0, sizeof(g.ids));
    memset(g.cq, 0, sizeof(g.cq));
    memset(g.cv, 0, sizeof(g.cv));
    g.kind = op.kind;
    g.m = op.m;
    g.nc = op.nc;
    g.angle = op.angle;
    if (op.m < 0 || op.m > QSV_MAX_TARGETS || op.nc < 0 || op.nc > QSV_MAX_CONTROLS) {
      set_error("op %d: unsupported target/control count", i);
      return QSV_EINVAL;
    }
    for (int j = 0; j < op.m; ++j) {
      g.targets[j] = op.targets[j];
      g.ids[j] = op.ids[j];
    }
    for (int j = 0; j < op.nc; ++j) {
      g.cq[j] = op.control_qubits[j];
      g.cv[j] = op.control_values[j];
    }
    if (op.kind == QSV_OP_DENSE) {
      const size_t D = (size_t)1 << op.m;
      if (!op.data) {
        set_error("op %d: dense gate without a matrix", i);
        return QSV_EINVAL;
      }
      g.data.resize(D * D);
      memcpy(g.data.data(), op.data, D * D * sizeof(Cplx));
    } else if (op.kind == QSV_OP_SPARSE) {
      if (op.nnz < 0 || (op.nnz > 0 && (!op.data || !op.sp_rows || !op.sp_cols))) {
        set_error("op %d: sparse gate without entries", i);
        return QSV_EINVAL;
      }
      g.data.resize(op.nnz);
      if (op.nnz) memcpy(g.data.data(), op.data, op.nnz * sizeof(Cplx));
      g.sp_rows.assign(op.sp_rows, op.sp_rows + op.nnz);
      g.sp_cols.assign(op.sp_cols, op.sp_cols + op.nnz);
    } else if (op.kind == QSV_OP_DIAG) {
      const size_t D = (size_t)1 << op.m;
      if (!op.data) {
        set_error("op %d: diagonal gate without entries", i);
        return QSV_EINVAL;
      }
      g.data.resize(D);
      memcpy(g.data.data(), op.data, D * sizeof(Cplx));
    }
    int rc = validate_gate(n, g);
    if (rc) {
      std::string msg = qsv_last_error();
      set_error("op %d: %s", i, msg.c_str());
      return rc;
    }
    g = canonicalize(g);
    if (g.nc < 0) continue;  // identity
    gates.push_back(g);
  }
  return QSV_OK;
}

extern "C" {

int qsv_plan_stats(int n, const qsv_op* ops, int nops, const qsv_plan_opts* opts,
                   qsv_program_stats* out) {
  if (!out || n < 1 || n > 40 || nops < 0 || (nops > 0 && !ops)) {
    set_error("bad plan arguments");
    return QSV_EINVAL;
  }
  qsv_plan_opts o{1, 0, 1, 1, 1, 1, 0};
  if (opts) o = *opts;
  std::vector<GateDesc> gates;
  int rc = convert_ops(n, ops, nops, gates);
  if (rc) return rc;
  std::vector<Step> steps;
  std::vector<TilePlan> tiles;
  std::vector<char> payload;
  memset(out, 0, sizeof(*out));
  out->num_ops_in = nops;
  return plan_program(n, gates, o, steps, tiles, payload, out);
}

int qsv_program_create(int n, const qsv_op* ops, int nops, const qsv_plan_opts* opts,
                       qsv_program** out) {
  if (!out) {
    set_error("null output pointer");
    return QSV_EINVAL;
  }
  *out = nullptr;
  if (n < 1 || n > 40 || nops < 0 || (nops > 0 && !ops)) {
    set_error("bad program arguments");
    return QSV_EINVAL;
  }
  qsv_plan_opts o{1, 0, 1, 1, 1, 1, 0};
  if (opts) o = *opts;
  std::vector<GateDesc> gates;
  int rc0 = convert_ops(n, ops, nops, gates);
  if (rc0) return rc0;

  qsv_program* p = new qsv_program();
  p->n = n;
  p->opts = o;
  memset(&p->stats, 0, sizeof(p->stats));
  p->stats.num_ops_in = nops;

  int rc = plan_program(n, gates, o, p->steps, p->tiles, p->host_payload, &p->stats);
  if (rc) {
    delete p;
    return rc;
  }
  p->payload_bytes = p->host_payload.size();
  int dev = 0;
  cudaGetDevice(&dev);
  rc = upload_payload(p, dev);
  if (rc) {
    delete p;
    return rc;
  }
  p->device = dev;
  // jit 2: compile now; jit 1: now only if every pass is already loaded or
  // its structure was planned before (a parametric recompile, a repeated segment)
  // (structure seen before, e.g. a VQE recompile with new angles)
  bool need_jit = false;  // passes the interpreter cannot run
  for (const TilePlan& tp : p->tiles) need_jit = need_jit || tp.jit_only;
  if (o.jit == 2 || need_jit || (o.jit == 1 && (jit_all_cached(p) || jit_all_seen(p)))) {
    rc = jit_prepare(p);
    if (rc) {
      qsv_program_destroy(p);
      return rc;
    }
  }
  *out = p;
  return QSV_OK;
}

int qsv_program_run(qsv_program* p, qsv_state* st) {
  if (!p || !st) {
    set_error("null handle");
    return QSV_EINVAL;
  }
  if (p->n != st->n) {
    set_error("state and circuit qubit counts differ (%d vs %d)", st->n, p->n);
    return QSV_EINVAL;
  }
  DeviceGuard dg(st->device);
  if (p->payload_device != st->device && !p->host_payload.empty()) {
    drop_graph(p);
    const int rc = upload_payload(p, st->device);
    if (rc) return rc;
  }
  if (p->payload_ready) QSV_TRY(cudaStreamWaitEvent(st->stream, p->payload_ready, 0));
  p->last_stream = st->stream;
  // the second run compiles the generated pass kernels (a program that runs
  // once never pays for NVRTC) -- before the graph capture, so the graph
  // holds them
  if (p->opts.jit && p->runs >= 1 && !p->jit_tried) {
    const int rc = jit_prepare(p);
    if (rc) return rc;
    drop_graph(p);
  }
  // the first run launches directly: a program that runs once (a recompile
  // after set_parameter) never pays for graph capture + instantiation
  if (!p->opts.use_graph || p->steps.empty() || p->runs++ == 0)
    return launch_steps(p, st->amps, st->stream, st->sm_limit, st->tile_ctr);
  // the graph bakes in the amplitude buffer AND the state's work counter: a
  // new state may reuse a freed amplitude block while its counter lives
  // elsewhere, so both pointers are part of the key
  if (!(p->gexec && p->graph_amps == st->amps && p->graph_ctr == st->tile_ctr &&
        p->graph_stream == st->stream &&
        p->device == st->device && p->graph_sm_limit == st->sm_limit)) {
    drop_graph(p);
    // capture on a private stream (the legacy stream cannot be captured)
    cudaStream_t cap;
    QSV_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      cudaStreamDestroy(cap);
      return cuda_fail(e, "cudaStreamBeginCapture");
    }
    int rc = launch_steps(p, st->amps, cap, st->sm_limit, st->tile_ctr);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&p->gexec, g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      return cuda_fail(e, "cudaGraphInstantiate");
    }
    p->graph = g;
    p->graph_amps = st->amps;
    p->graph_ctr = st->tile_ctr;
    p->graph_stream = st->stream;
    p->graph_sm_limit = st->sm_limit;
    p->device = st->device;
  }
  QSV_TRY(cudaGraphLaunch(p->gexec, st->stream));
  return QSV_OK;
}

int qsv_program_run_fixed(qsv_program* p, qsv_state* st, uint64_t mask, uint64_t value) {
  if (!p || !st) {
    set_error("null handle");
    return QSV_EINVAL;
  }
  if (p->n != st->n) {
    set_error("state and circuit qubit counts differ (%d vs %d)", st->n, p->n);
    return QSV_EINVAL;
  }
  if ((st->n < 64 && (mask >> st->n) != 0) || (value & ~mask) != 0) {
    set_error("fixed mask / value outside the state's qubits");
    return QSV_EINVAL;
  }
  for (const Step& s : p->steps) {
    if (s.type == 0) {
      set_error("program has per-gate kernels; only tile passes can run on a block");
      return QSV_EUNSUPPORTED;
    }
    for (int q : p->tiles[s.tile].qubits)
      if ((mask >> q) & 1) {
        set_error("fixed qubit %d is a tile qubit (plan with outer_mask)", q);
        return QSV_EINVAL;
      }
  }
  DeviceGuard dg(st->device);
  if (p->payload_device != st->device && !p->host_payload.empty()) {
    drop_graph(p);
    const int rc = upload_payload(p, st->device);
    if (rc) return rc;
  }
  if (p->opts.jit && p->runs++ >= 1 && !p->jit_tried) {
    const int rc = jit_prepare(p);
    if (rc) return rc;
  }
  if (p->payload_ready) QSV_TRY(cudaStreamWaitEvent(st->stream, p->payload_ready, 0));
  p->last_stream = st->stream;
  return launch_steps(p, st->amps, st->stream, st->sm_limit, st->tile_ctr, mask, value);
}

int qsv_program_stats_get(const qsv_program* p, qsv_program_stats* out) {
  if (!p || !out) {
    set_error("null handle");
    return QSV_EINVAL;
  }
  *out = p->stats;
  return QSV_OK;
}

int qsv_program_destroy(qsv_program* p) {
  if (!p) return QSV_OK;
  drop_graph(p);
  // freed in the order of the stream the program last ran on (pooled block)
  if (p->dev_payload) {
    DeviceGuard dg(p->payload_device);
    dev_free(p->dev_payload, p->payload_bytes, p->last_stream);
  }
  if (p->payload_ready) cudaEventDestroy(p->payload_ready);
  delete p;
  return QSV_OK;
}

}  // extern "C"
