// toy_bindings.cpp — END-TO-END TEST HARNESS: pybind11 module `_sfi_toy` over
// libsfi_toy.so (harness/engine.cpp): the reference's toy decoder and request
// loop (ToyModel, run_request, run_dense; proj/bindings/module.cpp:172-246)
// with the B200 hot path inside. Not part of the product package; imported by
// tests/test_engine.py through harness/__init__.py. Shared types (ModelSpec,
// configs, StepRecord) come from the product module `_sfi_b200`.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "sfi_b200.hpp"
#include "sfi_toy.hpp"

namespace py = pybind11;
using namespace sfi;

PYBIND11_MODULE(_sfi_toy, m) {
  m.doc() = "SFI toy decoder + request loop over the B200 hot path (test harness)";
  py::module_::import("paper_2603_12038_b200._sfi_b200");  // ModelSpec, configs, StepRecord, SfiError
  py::class_<ToyModel>(m, "ToyModel")
      .def_static("random", &ToyModel::random, py::arg("spec"), py::arg("seed"))
      .def("spec", &ToyModel::spec)
      .def("weight_checksum", [](const ToyModel& t) {
        // order-fixed sum over every weight (identity check against the reference's ToyModel::random)
        double acc = 0.0;
        auto add = [&](const std::vector<double>& v) { for (double x : v) acc += x; };
        add(t.embedding().v);
        for (int l = 0; l < t.spec().n_layers; ++l) {
          const auto& lw = t.layer(l);
          for (const auto* w : {&lw.wq, &lw.wk, &lw.wv, &lw.wo, &lw.w_gate, &lw.w_up, &lw.w_down}) add(w->v);
        }
        add(t.lm_head().v);
        return acc;
      });
  py::class_<RunOptions>(m, "RunOptions")
      .def(py::init<>())
      .def_readwrite("collect_logits", &RunOptions::collect_logits)
      .def_readwrite("capture_selected", &RunOptions::capture_selected);
  py::class_<RequestResult>(m, "RequestResult")
      .def_readonly("tokens", &RequestResult::tokens)
      .def_readonly("log", &RequestResult::log)
      .def_readonly("step_logits", &RequestResult::step_logits)
      .def_readonly("total_flops", &RequestResult::total_flops)
      .def_readonly("total_kv_reads", &RequestResult::total_kv_reads)
      .def_readonly("dense_equiv_reads", &RequestResult::dense_equiv_reads)
      .def_readonly("fast_retention", &RequestResult::fast_retention)
      .def_readonly("selected_per_step", &RequestResult::selected_per_step);
  py::class_<DenseResult>(m, "DenseResult")
      .def_readonly("tokens", &DenseResult::tokens)
      .def_readonly("step_logits", &DenseResult::step_logits)
      .def_readonly("total_kv_reads", &DenseResult::total_kv_reads)
      .def_readonly("total_flops", &DenseResult::total_flops);
  m.def("argmax_token", &argmax_token, py::arg("logits"));
  m.def("run_request", &run_request, py::arg("model"), py::arg("prompt"), py::arg("limits"), py::arg("trigger"),
        py::arg("selector"), py::arg("max_new"), py::arg("opts") = RunOptions{},
        py::call_guard<py::gil_scoped_release>());
  m.def("run_dense", &run_dense, py::arg("model"), py::arg("prompt"), py::arg("max_new"),
        py::call_guard<py::gil_scoped_release>());

}
