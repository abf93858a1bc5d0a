// cw_jit.cu -- run-time compiled fused-kernel instances (NVRTC, sm_100a).
//
// The fused frame kernel (cw_frame.cuh) is a template over the geometry
// (KX, KY, KZ, BX, BY) and the unrolled lag count NL; the library ships the
// default geometry and the SURVEY §8d C5 sweep precompiled (cw_inst.cuh).
// Every other geometry the fused kernel supports (K <= MAXK, lag grids of
// <= MAXL entries, shared memory within the 227 KB per CTA) is compiled on
// first use by NVRTC from the same headers, cached as a cubin keyed by the
// geometry and a hash of the kernel sources, and loaded with
// cudaLibraryLoadData.  Parameters beyond the fused kernel's limits run the
// runtime-geometry kernels (cw_generic.cu).  NVRTC is resolved with dlopen:
// without it the library still loads and those geometries take the
// runtime-geometry path.
//
// Cache lookup order: $CW_JIT_CACHE, then <package>/jit_cache (cubins
// prebuilt by __graft_entry__.build(), travelling with the tree), then
// $HOME/.cache/cw_b200_jit; new cubins are written to the first writable one
// of $CW_JIT_CACHE and $HOME/.cache/cw_b200_jit.
#include "cw_inst.cuh"
#include "cw_jit.cuh"

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace cwb {
namespace {

struct Nvrtc {
    bool ok = false;
    int (*create)(void **, const char *, const char *, int, const char *const *, const char *const *) = nullptr;
    int (*destroy)(void **) = nullptr;
    int (*add_name)(void *, const char *) = nullptr;
    int (*compile)(void *, int, const char *const *) = nullptr;
    int (*log_size)(void *, size_t *) = nullptr;
    int (*log)(void *, char *) = nullptr;
    int (*cubin_size)(void *, size_t *) = nullptr;
    int (*cubin)(void *, char *) = nullptr;
    int (*lowered)(void *, const char *, const char **) = nullptr;
    int (*version)(int *, int *) = nullptr;
};

Nvrtc &nvrtc()
{
    static Nvrtc n = [] {
        Nvrtc r;
        void *h = nullptr;
        // the toolkit's NVRTC first (the one nvcc built the library with),
        // not whichever libnvrtc.so.12 the process already loaded (torch)
        for (const char *name : {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)))
                break;
        if (!h)
            return r;
        auto sym = [&](auto &fp, const char *s) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, s)); return fp != nullptr; };
        r.ok = sym(r.create, "nvrtcCreateProgram") && sym(r.destroy, "nvrtcDestroyProgram") &&
               sym(r.add_name, "nvrtcAddNameExpression") && sym(r.compile, "nvrtcCompileProgram") &&
               sym(r.log_size, "nvrtcGetProgramLogSize") && sym(r.log, "nvrtcGetProgramLog") &&
               sym(r.cubin_size, "nvrtcGetCUBINSize") && sym(r.cubin, "nvrtcGetCUBIN") &&
               sym(r.lowered, "nvrtcGetLoweredName") && sym(r.version, "nvrtcVersion");
        return r;
    }();
    return n;
}

std::string dir_of_library()
{
    Dl_info info;
    if (dladdr(reinterpret_cast<void *>(&jit_instance), &info) && info.dli_fname) {
        std::string p = info.dli_fname;
        const size_t k = p.rfind('/');
        return k == std::string::npos ? std::string(".") : p.substr(0, k);
    }
    return ".";
}

std::string csrc_dir()
{
    if (const char *e = std::getenv("CW_CSRC"))
        return e;
    return dir_of_library() + "/csrc";
}

bool read_file(const std::string &path, std::string *out)
{
    std::ifstream f(path, std::ios::binary);
    if (!f)
        return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    *out = ss.str();
    return true;
}

unsigned long long fnv1a(const std::string &s, unsigned long long h = 1469598103934665603ull)
{
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

struct Entry {
    std::string cubin, frame_name, naive_name;
};

bool load_entry(const std::string &path, Entry *e)
{
    std::string blob;
    if (!read_file(path, &blob))
        return false;
    std::istringstream in(blob);
    std::string magic, fn, nn, size;
    if (!std::getline(in, magic) || magic != "cw_b200_jit 1" || !std::getline(in, fn) || !std::getline(in, nn) ||
        !std::getline(in, size))
        return false;
    const size_t n = std::strtoull(size.c_str(), nullptr, 10), off = (size_t)in.tellg();
    if (off + n != blob.size())
        return false;
    e->cubin = blob.substr(off);
    e->frame_name = fn;
    e->naive_name = nn;
    return true;
}

bool store_entry(const std::string &dir, const std::string &file, const Entry &e)
{
    mkdir(dir.c_str(), 0755);
    const std::string tmp = dir + "/" + file + ".tmp" + std::to_string((long long)getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f)
            return false;
        f << "cw_b200_jit 1\n" << e.frame_name << "\n" << e.naive_name << "\n" << e.cubin.size() << "\n";
        f.write(e.cubin.data(), (std::streamsize)e.cubin.size());
        if (!f)
            return false;
    }
    return std::rename(tmp.c_str(), (dir + "/" + file).c_str()) == 0;
}

bool compile(int kx, int ky, int kz, int bx, int by, int nl, Entry *e, std::string *err)
{
    Nvrtc &nv = nvrtc();
    if (!nv.ok) {
        *err = "NVRTC not available";
        return false;
    }
    char geo[128], fname[192], nname[160];
    snprintf(geo, sizeof geo, "cwb::Geo<%d, %d, %d, %d, %d>", kx, ky, kz, bx, by);
    snprintf(fname, sizeof fname, "cwb::cw_frame_kernel<%s, %d>", geo, nl);
    snprintf(nname, sizeof nname, "cwb::cw_naive_kernel<%s>", geo);
    const char *src = "#include \"cw_frame.cuh\"\n#include \"cw_naive.cuh\"\n";
    void *prog = nullptr;
    if (nv.create(&prog, src, "cw_jit_instance.cu", 0, nullptr, nullptr) != 0) {
        *err = "nvrtcCreateProgram failed";
        return false;
    }
    nv.add_name(prog, fname);
    nv.add_name(prog, nname);
    const std::string inc = "-I" + csrc_dir();
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                          inc.c_str(), "-I/usr/local/cuda/include"};
    const int rc = nv.compile(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    if (rc != 0) {
        size_t n = 0;
        nv.log_size(prog, &n);
        std::string log(n, '\0');
        nv.log(prog, &log[0]);
        *err = "NVRTC compile failed: " + log.substr(0, 2000);
        nv.destroy(&prog);
        return false;
    }
    size_t n = 0;
    nv.cubin_size(prog, &n);
    e->cubin.assign(n, '\0');
    nv.cubin(prog, &e->cubin[0]);
    const char *lf = nullptr, *ln = nullptr;
    nv.lowered(prog, fname, &lf);
    nv.lowered(prog, nname, &ln);
    e->frame_name = lf ? lf : "";
    e->naive_name = ln ? ln : "";
    nv.destroy(&prog);
    return !e->frame_name.empty() && !e->naive_name.empty();
}

std::string source_key(int kx, int ky, int kz, int bx, int by, int nl)
{
    std::string a, b;
    read_file(csrc_dir() + "/cw_frame.cuh", &a);
    read_file(csrc_dir() + "/cw_naive.cuh", &b);
    int maj = 0, min = 0;
    if (nvrtc().ok)
        nvrtc().version(&maj, &min);
    char buf[160];
    snprintf(buf, sizeof buf, "g%d_%d_%d_%d_%d_nl%d_%016llx_nvrtc%d.%d.cubin", kx, ky, kz, bx, by, nl,
             fnv1a(b, fnv1a(a)), maj, min);
    return buf;
}

std::mutex g_mu;
std::map<std::string, LaunchFn> g_loaded;  // process-wide: libraries stay loaded

}  // namespace

bool jit_supported(int kx, int ky, int kz, int bx, int by, int nlx, int nly)
{
    if (kx > MAXK || ky > MAXK || nlx > MAXL || nly > MAXL)
        return false;
    const GeoSizes g = geo_sizes(kx, ky, kz, bx, by);
    return g.smem <= 232448 && g.naive_smem <= 232448 && g.threads <= 1024;
}

bool jit_instance(int kx, int ky, int kz, int bx, int by, int nl, LaunchFn *out, std::string *err)
{
    std::lock_guard<std::mutex> lock(g_mu);
    const std::string file = source_key(kx, ky, kz, bx, by, nl);
    auto it = g_loaded.find(file);
    if (it != g_loaded.end()) {
        *out = it->second;
        return true;
    }
    std::vector<std::string> dirs;
    if (const char *e = std::getenv("CW_JIT_CACHE"))
        dirs.push_back(e);
    dirs.push_back(dir_of_library() + "/jit_cache");
    const char *home = std::getenv("HOME");
    const std::string user = std::string(home ? home : "/tmp") + "/.cache/cw_b200_jit";
    dirs.push_back(user);
    Entry e;
    bool have = false;
    for (const std::string &d : dirs)
        if ((have = load_entry(d + "/" + file, &e)))
            break;
    if (!have) {
        if (!compile(kx, ky, kz, bx, by, nl, &e, err))
            return false;
        const char *ce = std::getenv("CW_JIT_CACHE");
        if (!(ce && store_entry(ce, file, e))) {
            mkdir((std::string(home ? home : "/tmp") + "/.cache").c_str(), 0755);
            store_entry(user, file, e);
        }
    }
    cudaLibrary_t lib;
    cudaKernel_t kf, kn;
    if (cudaLibraryLoadData(&lib, e.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&kf, lib, e.frame_name.c_str()) != cudaSuccess ||
        cudaLibraryGetKernel(&kn, lib, e.naive_name.c_str()) != cudaSuccess) {
        cudaGetLastError();
        *err = "cannot load the run-time compiled kernel";
        return false;
    }
    const GeoSizes g = geo_sizes(kx, ky, kz, bx, by);
    LaunchFn f{};
    f.kernel = reinterpret_cast<const void *>(kf);
    f.naive_kernel = reinterpret_cast<const void *>(kn);
    f.naive_smem = g.naive_smem;
    f.threads = g.threads;
    f.smem = g.smem;
    f.nsp = g.nsp;
    f.ntp = g.ntp;
    f.retp = g.retpp;
    f.nl = nl;
    f.pef_l2 = g.pef_l2;
    f.compact = g.compact;
    g_loaded[file] = f;
    *out = f;
    return true;
}

int jit_prebuild(int kx, int ky, int kz, int bx, int by, int nl, const char *dir, std::string *err)
{
    Entry e;
    const std::string file = source_key(kx, ky, kz, bx, by, nl);
    if (load_entry(std::string(dir) + "/" + file, &e))
        return 0;
    if (!compile(kx, ky, kz, bx, by, nl, &e, err))
        return -1;
    return store_entry(dir, file, e) ? 0 : -1;
}

}  // namespace cwb
